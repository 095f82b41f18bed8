// C-ABI runtime of the B200-native PilotANN GPU stage (include/pilotann.h).
// Validation → device replica (ELL subgraph, reduced vectors, FES pool grouped
// by cell) → per-search pipeline: H2D → a1 projection → a2/a4 FES → a5/a6
// traversal → a7 D2H [→ a8/a9 host stages].
#include "pilotann.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "host_stages.h"
#include "internal.h"

namespace {

thread_local std::string g_err;

pa_status fail(pa_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CU(expr)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) {                                                                 \
            return fail(e_ == cudaErrorMemoryAllocation ? PA_ENOMEM : PA_ECUDA, "%s: %s (%s:%d)", \
                        #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                      \
        }                                                                                        \
    } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    return cudaMalloc((void**)p, std::max<size_t>(1, count) * sizeof(T));
}

std::mutex g_reg_mu;
std::unordered_set<const void*> g_live;   // live handles (double destroy / use-after-destroy guard)

int threads_default(int req) {
    if (req > 0) return req;
    if (const char* s = std::getenv("PILOTANN_HOST_THREADS")) {
        int v = std::atoi(s);
        if (v > 0) return v;
    }
    return (int)std::max(1u, std::thread::hardware_concurrency());
}

template <class F>
void parallel_rows(int64_t n, F f) {
    int T = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), std::max<int64_t>(1, n / 65536 + 1));
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=]() { f(n * t / T, n * (t + 1) / T); });
    for (auto& x : th) x.join();
}

// Validate a CSR over n nodes: S:L183-186.  Returns 0 or an error message code.
pa_status check_csr(const int64_t* off, const int32_t* nb, int64_t n, int32_t max_degree, const char* what) {
    if (off[0] != 0) return fail(PA_EGRAPH, "%s: offsets[0] = %lld, expected 0", what, (long long)off[0]);
    std::atomic<int64_t> bad_row{-1};
    std::atomic<int> bad_kind{0};
    parallel_rows(n, [&](int64_t lo, int64_t hi) {
        std::vector<int32_t> tmp;
        for (int64_t u = lo; u < hi && bad_row.load() < 0; ++u) {
            int64_t a = off[u], b = off[u + 1];
            if (b < a) { bad_kind = 1; bad_row = u; return; }
            if (max_degree > 0 && b - a > max_degree) { bad_kind = 2; bad_row = u; return; }
            tmp.assign(nb + a, nb + b);
            for (int32_t v : tmp)
                if (v < 0 || v >= n) { bad_kind = 3; bad_row = u; return; }
                else if (v == u) { bad_kind = 4; bad_row = u; return; }
            std::sort(tmp.begin(), tmp.end());
            for (size_t i = 1; i < tmp.size(); ++i)
                if (tmp[i] == tmp[i - 1]) { bad_kind = 5; bad_row = u; return; }
        }
    });
    if (bad_row.load() >= 0) {
        static const char* kinds[] = {"", "offsets not monotone", "degree exceeds max_degree",
                                      "neighbour id out of range", "self-loop", "duplicate neighbour"};
        return fail(PA_EGRAPH, "%s: %s at node %lld", what, kinds[bad_kind.load()], (long long)bad_row.load());
    }
    return PA_OK;
}

// Level-1 visited-table size (slots = 2^this).  Tuned on C1 (gpurun t2/t3):
// 16-bit quotiented slots (ids < 2^24): 2^11 up to ef 64, 2^12 above (8 KB);
// 32-bit slots: 2^11 up to ef 128 (8 KB), 2^12 above.
int default_hash_log2(int ef, int64_t n) {
    if (n <= (1 << 24)) return ef <= 64 ? 11 : 12;
    return ef <= 128 ? 11 : 12;
}

}  // namespace

// ----------------------------------------------------------------------------
struct pa_index {
    static constexpr uint32_t kMagic = 0x50414e4eu;   // "PANN"
    uint32_t magic = kMagic;
    int device = 0;
    pa::DevIndex dev;
    std::vector<int64_t> h_sub_off;        // host copy of the subgraph for stage ②
    std::vector<int32_t> h_sub_nb;
    const int64_t* h_full_off = nullptr;   // borrowed (pa_attach_host)
    const int32_t* h_full_nb = nullptr;
    const float* h_rotated = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;                 // a7 handoff (D2H of candidates)
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};   // project | fes | traverse | refine
    std::vector<cudaEvent_t> pipe_done, pipe_copied;    // per sub-batch (stages ②③ pipeline)
    cudaEvent_t pipe_start = nullptr, pipe_end = nullptr;
    cudaEvent_t done_ev = nullptr;         // end of the last enqueued search (any stream)
    bool done_recorded = false;
    std::mutex mu;
    pa_stats stats{};
    bool events_pending = false;
    bool last_full_gpu = false;           // last search ran ②③ on the GPU (counters2 valid)
    // workspace
    int64_t ws_m = 0;
    int32_t ws_E = 0, ws_ef = 0, ws_k = 0;
    float *q = nullptr, *qp = nullptr, *qres = nullptr, *cand_d = nullptr, *out_d = nullptr;
    int32_t* counters2 = nullptr;          // [m][4] stages ②③ on the GPU: n_dist2, n_dist3, 0, status
    int32_t *cell = nullptr, *entries = nullptr, *cand_ids = nullptr, *out_ids = nullptr, *counters = nullptr,
            *work = nullptr, *perm = nullptr, *qoff = nullptr, *toff = nullptr;
    float* fes_scores = nullptr;
    uint64_t* spill = nullptr;
    int64_t spill_warps = 0;
    int32_t spill_log2 = 16;
    uint32_t epoch_base = 1;
    // pinned host staging for the host stages
    int64_t h_m = 0;
    int32_t h_ef = 0;
    int32_t *h_cand_ids = nullptr, *h_counters = nullptr;
    float *h_cand_d = nullptr, *h_qp = nullptr, *h_qres = nullptr;
};

namespace {

bool live(const pa_index* ix) {
    std::lock_guard<std::mutex> g(g_reg_mu);
    return ix && g_live.count(ix) && ix->magic == pa_index::kMagic;
}

void free_ws(pa_index* ix) {
    cudaFree(ix->q); cudaFree(ix->qp); cudaFree(ix->qres); cudaFree(ix->cand_d); cudaFree(ix->out_d);
    cudaFree(ix->cell); cudaFree(ix->entries); cudaFree(ix->cand_ids); cudaFree(ix->out_ids);
    cudaFree(ix->counters); cudaFree(ix->work); cudaFree(ix->perm); cudaFree(ix->qoff); cudaFree(ix->toff);
    cudaFree(ix->fes_scores);
    cudaFree(ix->counters2);
    ix->fes_scores = nullptr;
    ix->counters2 = nullptr;
    ix->q = ix->qp = ix->qres = ix->cand_d = ix->out_d = nullptr;
    ix->cell = ix->entries = ix->cand_ids = ix->out_ids = ix->counters = ix->work = nullptr;
    ix->perm = ix->qoff = ix->toff = nullptr;
    ix->ws_m = 0;
}

pa_status ensure_ws(pa_index* ix, int64_t m, int32_t E, int32_t ef, int32_t k) {
    if (m <= ix->ws_m && E <= ix->ws_E && ef <= ix->ws_ef && k <= ix->ws_k) return PA_OK;
    free_ws(ix);
    m = std::max<int64_t>(m, 1);
    E = std::max(E, ix->ws_E); ef = std::max(ef, ix->ws_ef); k = std::max(k, ix->ws_k);
    const auto& d = ix->dev;
    CU(dalloc(&ix->q, (size_t)m * d.dim));
    CU(dalloc(&ix->qp, (size_t)m * d.rdim_pad));
    CU(dalloc(&ix->qres, (size_t)m * std::max(1, d.dim - d.rdim)));
    CU(dalloc(&ix->cell, (size_t)m));
    CU(dalloc(&ix->entries, (size_t)m * E));
    CU(dalloc(&ix->cand_ids, (size_t)m * ef));
    CU(dalloc(&ix->cand_d, (size_t)m * ef));
    CU(dalloc(&ix->out_ids, (size_t)m * k));
    CU(dalloc(&ix->out_d, (size_t)m * k));
    CU(dalloc(&ix->counters, (size_t)m * 4));
    CU(dalloc(&ix->counters2, (size_t)m * 4));
    CU(dalloc(&ix->work, 4));
    CU(dalloc(&ix->perm, (size_t)m));
    CU(dalloc(&ix->qoff, (size_t)d.fes_r + 1));
    CU(dalloc(&ix->toff, (size_t)d.fes_r + 1));
    CU(dalloc(&ix->fes_scores, pa::fes_tc_scratch_floats(d, m)));
    ix->ws_m = m; ix->ws_E = E; ix->ws_ef = ef; ix->ws_k = k;
    return PA_OK;
}

pa_status ensure_spill(pa_index* ix, int64_t warps) {
    if (warps <= ix->spill_warps) return PA_OK;
    cudaFree(ix->spill);
    ix->spill = nullptr;
    ix->spill_warps = 0;
    size_t bytes = (size_t)warps * ((size_t)8 << ix->spill_log2);
    CU(cudaMalloc((void**)&ix->spill, bytes));
    CU(cudaMemset(ix->spill, 0, bytes));
    ix->spill_warps = warps;
    ix->epoch_base = 1;
    return PA_OK;
}

struct Resolved {
    int32_t stages, ef1, ef2, ef3, E, width, refine, hash_log2, threads, bloom_log2;
    uint32_t flags, check;
};

pa_status resolve(const pa_search_opts* o, int32_t k, int32_t ef, Resolved* r, int64_t n) {
    pa_search_opts z{};
    if (!o) o = &z;
    r->stages = o->stages ? o->stages : PA_STAGES_GPU;
    if (r->stages != PA_STAGES_GPU && r->stages != PA_STAGES_FULL && r->stages != PA_STAGES_FULL_GPU)
        return fail(PA_EINVAL, "bad stages %d", r->stages);
    if (k < 1) return fail(PA_EINVAL, "k = %d < 1", k);
    if (ef < k) return fail(PA_EINVAL, "ef = %d < k = %d", ef, k);
    r->ef1 = o->ef1 ? o->ef1 : ef;
    r->ef3 = o->ef3 ? o->ef3 : ef;
    r->ef2 = o->ef2 ? o->ef2 : std::max(k, ef / 2);
    r->E = o->entries ? o->entries : r->ef1;
    r->width = o->width ? o->width : 1;
    r->refine = o->refine_iters == 0 ? 2 : (o->refine_iters < 0 ? 0 : o->refine_iters);
    r->flags = o->flags;
    r->check = o->check_path;
    if (r->check & ~(uint32_t)(PA_CHECK_SIMT | PA_CHECK_WIDE_VISITED)) return fail(PA_EINVAL, "bad check_path %u", r->check);
    r->hash_log2 = o->hash_slots_log2 ? o->hash_slots_log2 : default_hash_log2(r->ef1, n);
    r->threads = threads_default(o->host_threads);
    r->bloom_log2 = o->bloom_log2;
    if (r->bloom_log2 != 0 && (r->bloom_log2 < 7 || r->bloom_log2 > 16))
        return fail(PA_EINVAL, "bloom_log2 = %d (0 or 7..16)", r->bloom_log2);
    // stage ① (and its FES entries) is bounded by the traversal kernels' 256-key lists;
    // the refinement stages ②③ keep up to 512 (the ef stage ③ needs for full-space
    // Recall@10 = 0.90 at 100M, DESIGN §3 reading R-ef)
    if (r->ef1 > 256) return fail(PA_EINVAL, "ef1 = %d > 256", r->ef1);
    if (r->ef2 > 512 || r->ef3 > 512) return fail(PA_EINVAL, "ef2/ef3 > 512");
    if (r->ef1 < 1 || r->ef2 < 1 || r->ef3 < 1 || r->E < 1 || r->E > 1024) return fail(PA_EINVAL, "bad ef/entries");
    if (r->stages == PA_STAGES_GPU && k > r->ef1) return fail(PA_EINVAL, "k = %d > ef1 = %d", k, r->ef1);
    if (r->stages != PA_STAGES_GPU && (k > r->ef3 || k > r->ef2)) return fail(PA_EINVAL, "k > ef2/ef3");
    if (r->width < 1 || r->width > 8) return fail(PA_EINVAL, "search width w = %d not in 1..8", r->width);
    if (r->width > 1 && r->bloom_log2 > 0)
        return fail(PA_ENOTSUP, "search width w > 1 uses the exact visited set (bloom_log2 must be 0)");
    if (r->hash_log2 < 5 || r->hash_log2 > 15) return fail(PA_EINVAL, "hash_slots_log2 = %d", r->hash_log2);
    return PA_OK;
}

// NEXT-f3: device copies of the full graph (ELL, −1 padded) and of X̂ (rows on a
// 128-B-aligned stride) from the arrays pa_attach_host borrowed; once per index.
pa_status ensure_full_device(pa_index* ix) {
    auto& d = ix->dev;
    if (d.xhat) return PA_OK;
    if (!ix->h_rotated || !ix->h_full_off) return fail(PA_ESTATE, "PA_STAGES_FULL_GPU requires pa_attach_host");
    const int64_t n = d.n;
    int64_t maxdeg = 0;
    for (int64_t u = 0; u < n; ++u) maxdeg = std::max<int64_t>(maxdeg, ix->h_full_off[u + 1] - ix->h_full_off[u]);
    if (maxdeg > 64) return fail(PA_ENOTSUP, "PA_STAGES_FULL_GPU: full-graph degree %lld > 64", (long long)maxdeg);
    const int w = maxdeg <= 32 ? 32 : 64;
    const int xs = (d.dim + 31) & ~31;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = (size_t)n * (w * 4 + (size_t)xs * 4);
    if (need + ((size_t)1 << 30) > fr) return fail(PA_ENOMEM, "PA_STAGES_FULL_GPU: %zu MB needed, %zu MB free", need >> 20, fr >> 20);
    int32_t* ell = nullptr;
    float* xh = nullptr;
    CU(dalloc(&ell, (size_t)n * w));
    if (dalloc(&xh, (size_t)n * xs) != cudaSuccess) { cudaFree(ell); return fail(PA_ENOMEM, "X̂ allocation"); }
    const int64_t chunk = 1 << 20;
    std::vector<int32_t> eb((size_t)std::min(chunk, n) * w);
    std::vector<float> xb((size_t)std::min(chunk, n) * xs);
    for (int64_t s0 = 0; s0 < n; s0 += chunk) {
        const int64_t s1 = std::min(n, s0 + chunk);
        parallel_rows(s1 - s0, [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) {
                const int64_t u = s0 + i, a0 = ix->h_full_off[u], a1 = ix->h_full_off[u + 1];
                for (int j = 0; j < w; ++j) eb[(size_t)i * w + j] = a0 + j < a1 ? ix->h_full_nb[a0 + j] : -1;
                std::memcpy(&xb[(size_t)i * xs], ix->h_rotated + u * d.dim, sizeof(float) * d.dim);
                for (int j = d.dim; j < xs; ++j) xb[(size_t)i * xs + j] = 0.f;
            }
        });
        CU(cudaMemcpy(ell + s0 * w, eb.data(), sizeof(int32_t) * (s1 - s0) * w, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(xh + s0 * xs, xb.data(), sizeof(float) * (s1 - s0) * xs, cudaMemcpyHostToDevice));
    }
    d.full_ell = ell; d.full_w = w; d.xhat = xh; d.xstride = xs;
    return PA_OK;
}

// Enqueue a1..a6 on stream s for device queries q → out ids/dists.
pa_status enqueue_gpu_stage(pa_index* ix, const float* d_q, int64_t m, int32_t k, const Resolved& r,
                            int32_t* d_out_ids, float* d_out_d, const pa_debug* dbg, bool want_qres,
                            cudaStream_t s, int64_t row0 = 0) {
    pa_status st = ensure_ws(ix, row0 + m, r.E, r.ef1, k);
    if (st != PA_OK) return st;
    const auto& dd = ix->dev;
    if (r.stages == PA_STAGES_FULL_GPU && (!dd.xhat || !dd.full_ell))
        return fail(PA_ESTATE, "stages 2-3 on the GPU need the device copy of the full graph and X-hat");
    // Every search on this index shares its workspace (work counter, candidate and
    // spill buffers): a search enqueued on another stream first waits for the end
    // of the previous one, so calls serialise on the device as well as on the mutex.
    if (ix->done_recorded) CU(cudaStreamWaitEvent(s, ix->done_ev, 0));
    pa::SearchArgs a;
    a.m = m; a.k = k; a.ef = r.ef1; a.E = r.E; a.flags = r.flags; a.hash_log2 = r.hash_log2;
    a.bloom_log2 = r.bloom_log2;
    a.wide_visited = (r.check & PA_CHECK_WIDE_VISITED) != 0;
    a.width = r.width;
    if (a.bloom_log2 > 0 && dd.ell_w != 32) return fail(PA_ENOTSUP, "bloom visited set needs max_degree <= 32");
    a.q = d_q; a.qp = ix->qp + row0 * dd.rdim_pad;
    a.qres = want_qres ? ix->qres + row0 * std::max(1, dd.dim - dd.rdim) : nullptr;
    a.cell = (dbg && dbg->cell) ? dbg->cell : ix->cell + row0;
    a.entries = (dbg && dbg->entries) ? dbg->entries : ix->entries + row0 * r.E;
    a.cand_ids = (dbg && dbg->cand_ids) ? dbg->cand_ids : ix->cand_ids + row0 * r.ef1;
    a.cand_d = (dbg && dbg->cand_dists) ? dbg->cand_dists : ix->cand_d + row0 * r.ef1;
    a.counters = (dbg && dbg->counters) ? dbg->counters : ix->counters + row0 * 4;
    a.out_ids = d_out_ids; a.out_d = d_out_d;
    a.work = ix->work;
    a.perm = ix->perm; a.qoff = ix->qoff; a.toff = ix->toff; a.fes_scores = ix->fes_scores;
    if (dbg && dbg->trace_cap > 0 && dbg->trace_expand && dbg->trace_visit && dbg->trace_nexp && dbg->trace_nvis) {
        a.trace_cap = dbg->trace_cap; a.trace_expand = dbg->trace_expand; a.trace_visit = dbg->trace_visit;
        a.trace_nexp = dbg->trace_nexp; a.trace_nvis = dbg->trace_nvis;
    }
    int maxw = pa::traverse_max_warps(ix->dev, a);
    if (maxw <= 0) return fail(PA_ENOTSUP, "traversal does not fit on an SM (ef=%d, hash_log2=%d)", r.ef1, r.hash_log2);
    int64_t gridw = std::min<int64_t>(maxw, ((m + 3) / 4) * 4);
#ifndef PA_WAVE_BALANCE_PCT
#define PA_WAVE_BALANCE_PCT 0          // balance the persistent grid's waves if that drops ≤ this % of its warps
#endif
    if (PA_WAVE_BALANCE_PCT > 0 && m > maxw) {
        // per-query work is ≈ ef expansions whatever the query (n_exp ≈ ef), so the grid runs
        // in near-discrete waves of gridw queries; a last wave of m mod gridw queries leaves
        // most warps idle — spread m over the same number of waves with fewer warps instead
        const int64_t waves = (m + maxw - 1) / maxw;
        const int64_t bal = ((m + waves - 1) / waves + 3) / 4 * 4;
        if (bal * 100 >= (int64_t)maxw * (100 - PA_WAVE_BALANCE_PCT)) gridw = bal;
    }
    st = ensure_spill(ix, gridw);
    if (st != PA_OK) return st;
    if ((uint64_t)ix->epoch_base + (uint64_t)m + 1 >= 0xffffffffull) {
        CU(cudaMemsetAsync(ix->spill, 0, (size_t)ix->spill_warps * ((size_t)8 << ix->spill_log2), s));
        ix->epoch_base = 1;
    }
    a.spill = ix->spill; a.spill_log2 = ix->spill_log2; a.spill_warps = ix->spill_warps;
    a.epoch_base = ix->epoch_base;
    ix->epoch_base += (uint32_t)m + 1;

    int launches = 0;
    CU(cudaEventRecord(ix->ev[0], s));
    const bool force_simt = (r.check & PA_CHECK_SIMT) != 0;   // test hook: the SIMT cross-check kernels
    if (!force_simt && pa::project_tc_supported(ix->dev, a.qres != nullptr)) {
        launches += pa::launch_project_tc(ix->dev, a, s);
        a.cell_ready = true;
    } else {
        launches += pa::launch_project(ix->dev, a, s);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(ix->ev[1], s));
    if (a.cell_ready && !force_simt && !(a.flags & PA_NO_FES) && pa::fes_tc_supported(ix->dev, a.E))
        launches += pa::launch_fes_tc(ix->dev, a, s);
    else
        launches += pa::launch_fes(ix->dev, a, s);
    CU(cudaGetLastError());
    CU(cudaEventRecord(ix->ev[2], s));
    launches += pa::launch_traverse(ix->dev, a, (int)gridw, s);
    CU(cudaGetLastError());
    CU(cudaEventRecord(ix->ev[3], s));
    if (r.stages == PA_STAGES_FULL_GPU) {                   // NEXT-f3: ②③ on the GPU
        pa::Refine23 f;
        f.m = m; f.k = k; f.ef1 = r.ef1; f.ef2 = r.ef2; f.ef3 = r.ef3; f.refine_iters = r.refine; f.flags = r.flags;
        f.width = r.width;
        f.D = dd.dim; f.dp = dd.rdim; f.qlen = (dd.dim + 3) & ~3; f.qp = a.qp; f.qp_stride = dd.rdim_pad;
        f.qres = a.qres; f.cand = a.cand_ids;
        f.sub_ell = dd.ell; f.sub_w = dd.ell_w; f.full_ell = dd.full_ell; f.full_w = dd.full_w;
        f.xhat = dd.xhat; f.xstride = dd.xstride;
        f.hash_log2 = dd.n <= (1 << 24) ? 12 : 11;        // ②③ visit ~20× ef ids: 8-KB smem table per query
        f.work = ix->work; f.out_ids = d_out_ids; f.out_d = d_out_d;
        f.counters = ix->counters2 ? ix->counters2 + row0 * 4 : nullptr;
        const int fw = pa::refine_max_warps(ix->dev, f);
        if (fw <= 0) return fail(PA_ENOTSUP, "stage 2-3 kernel does not fit on an SM");
        const int64_t fgw = std::min<int64_t>(fw, ((m + 3) / 4) * 4);
        st = ensure_spill(ix, fgw);
        if (st != PA_OK) return st;
        f.spill = ix->spill; f.spill_log2 = ix->spill_log2;
        launches += pa::launch_refine(ix->dev, f, (int)fgw, s);
        CU(cudaGetLastError());
    }
    CU(cudaEventRecord(ix->ev[4], s));
    CU(cudaEventRecord(ix->done_ev, s));
    ix->done_recorded = true;
    ix->events_pending = true;
    ix->last_full_gpu = r.stages == PA_STAGES_FULL_GPU;
    ix->stats = pa_stats{};
    ix->stats.queries = m;
    ix->stats.kernel_launches = launches;
    return PA_OK;
}

void collect_event_times(pa_index* ix) {
    if (!ix->events_pending) return;
    cudaEventSynchronize(ix->ev[4]);
    float t01 = 0, t12 = 0, t23 = 0, t34 = 0, t04 = 0;
    cudaEventElapsedTime(&t01, ix->ev[0], ix->ev[1]);
    cudaEventElapsedTime(&t12, ix->ev[1], ix->ev[2]);
    cudaEventElapsedTime(&t23, ix->ev[2], ix->ev[3]);
    cudaEventElapsedTime(&t34, ix->ev[3], ix->ev[4]);
    cudaEventElapsedTime(&t04, ix->ev[0], ix->ev[4]);
    ix->stats.ms_project = t01; ix->stats.ms_fes = t12; ix->stats.ms_traverse = t23; ix->stats.ms_refine = t34;
    ix->stats.ms_total_gpu = t04;
    ix->events_pending = false;
}

pa_status ensure_pipe_events(pa_index* ix, int64_t nb) {
    while ((int64_t)ix->pipe_done.size() < nb) {
        cudaEvent_t a, b;
        CU(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        ix->pipe_done.push_back(a);
        ix->pipe_copied.push_back(b);
    }
    if (!ix->pipe_start) {
        CU(cudaEventCreate(&ix->pipe_start));
        CU(cudaEventCreate(&ix->pipe_end));
    }
    return PA_OK;
}

pa_status ensure_host_ws(pa_index* ix, int64_t m, int32_t ef) {
    if (m <= ix->h_m && ef <= ix->h_ef) return PA_OK;
    cudaFreeHost(ix->h_cand_ids); cudaFreeHost(ix->h_cand_d); cudaFreeHost(ix->h_qp); cudaFreeHost(ix->h_qres);
    cudaFreeHost(ix->h_counters);
    ix->h_cand_ids = nullptr; ix->h_cand_d = ix->h_qp = ix->h_qres = nullptr; ix->h_counters = nullptr;
    ix->h_m = 0;
    const auto& d = ix->dev;
    CU(cudaMallocHost((void**)&ix->h_cand_ids, sizeof(int32_t) * m * ef));
    CU(cudaMallocHost((void**)&ix->h_cand_d, sizeof(float) * m * ef));
    CU(cudaMallocHost((void**)&ix->h_qp, sizeof(float) * m * d.rdim_pad));
    CU(cudaMallocHost((void**)&ix->h_qres, sizeof(float) * m * std::max(1, d.dim - d.rdim)));
    CU(cudaMallocHost((void**)&ix->h_counters, sizeof(int32_t) * m * 4));
    ix->h_m = m; ix->h_ef = ef;
    return PA_OK;
}

// The replica's device arrays in a fixed order (pa_replica_buffers): pointer slot + bytes.
void replica_list(pa::DevIndex& d, std::vector<std::pair<void**, size_t>>& L) {
    const size_t n = (size_t)d.n, r = (size_t)d.fes_r, dps = (size_t)d.rdim_pad, D = (size_t)d.dim;
    auto add = [&](auto** p, size_t bytes) { L.emplace_back(reinterpret_cast<void**>(p), bytes); };
    add(&d.basis, D * D * 4);
    if (d.reduced_h) add(&d.reduced_h, n * d.rstride_h * 2);
    else add(&d.reduced, n * d.rstride * 4);
    add(&d.ell, n * d.ell_w * 4);
    add(&d.centroids, r * dps * 4);
    add(&d.cell_off, (r + 1) * 4);
    add(&d.pool_ids, (size_t)d.pool_n * 4);
    add(&d.pool_vec, (size_t)d.pool_n * dps * 4);
    add(&d.pool_norm, (size_t)d.pool_n * 4);
    add(&d.pool_img, (size_t)d.pool_chunks * ((dps + 31) / 32) * 2 * 4096 * 4);
    add(&d.chunk_off, (r + 1) * 4);
    add(&d.proj_img, ((D + 31) / 32) * 2 * (size_t)d.proj_nb * 32 * 4);
    add(&d.cent_norm, r * 4);
    if (d.xhat) {
        add(&d.full_ell, n * d.full_w * 4);
        add(&d.xhat, n * d.xstride * 4);
    }
}

}  // namespace

// ============================================================================ ABI
extern "C" {

const char* pa_last_error(void) { return g_err.c_str(); }
const char* pa_version(void) { return "pilotann-b200 0.1 (sm_100a)"; }

pa_status pa_build(const pa_build_params* p, pa_index** out) {
    g_err.clear();
    if (!p || !out) return fail(PA_EINVAL, "null argument");
    *out = nullptr;
    if (!p->sub_offsets || !p->reduced || !p->basis || !p->fes_centroids || !p->fes_cell_off || !p->fes_pool_ids)
        return fail(PA_EINVAL, "null input array");
    if (p->n <= 0 || p->n >= (1ll << 31)) return fail(PA_EINVAL, "n = %lld out of range", (long long)p->n);
    if (p->sub_offsets[p->n] > 0 && !p->sub_neighbors) return fail(PA_EINVAL, "null sub_neighbors");
    if (p->dim <= 0 || p->rdim <= 0 || p->rdim > p->dim) return fail(PA_EINVAL, "bad dims D=%d d'=%d", p->dim, p->rdim);
    if (p->dim > 4096) return fail(PA_EINVAL, "dim %d > 4096", p->dim);
    if (p->max_degree < 1 || p->max_degree > 64) return fail(PA_EINVAL, "max_degree %d not in 1..64", p->max_degree);
    if (p->metric != PA_L2 && p->metric != PA_IP) return fail(PA_EINVAL, "bad metric %d", p->metric);
    if (p->fes_r < 1 || p->fes_r > 1024) return fail(PA_EINVAL, "fes_r %d not in 1..1024", p->fes_r);
    if (p->reduced_stride != 0 && p->reduced_stride < p->rdim)
        return fail(PA_EINVAL, "reduced_stride %lld < rdim %d", (long long)p->reduced_stride, p->rdim);
    const int64_t n = p->n;
    const int D = p->dim, dp = p->rdim;
    int64_t rsin = p->reduced_stride ? p->reduced_stride : dp;    // input row stride of `reduced`
    // ---- graph and subgraph invariants
    pa_status st = check_csr(p->sub_offsets, p->sub_neighbors, n, p->max_degree, "subgraph");
    if (st != PA_OK) return st;
    std::vector<uint8_t> member(n);
    for (int64_t u = 0; u < n; ++u) {
        bool deg = p->sub_offsets[u + 1] > p->sub_offsets[u];
        member[u] = p->member_flags ? (p->member_flags[u] != 0) : deg;
        if (!member[u] && deg) return fail(PA_EGRAPH, "non-member %lld has out-edges", (long long)u);
    }
    for (int64_t e = 0; e < p->sub_offsets[n]; ++e)
        if (!member[p->sub_neighbors[e]])
            return fail(PA_EGRAPH, "edge into non-member %d", p->sub_neighbors[e]);
    // ---- basis orthonormal and finite
    for (int64_t i = 0; i < (int64_t)D * D; ++i)
        if (!std::isfinite(p->basis[i])) return fail(PA_EINVAL, "non-finite basis entry %lld", (long long)i);
    {
        double worst = 0;
        std::vector<double> col((size_t)D * D);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) col[(size_t)j * D + i] = p->basis[(size_t)i * D + j];
        for (int a = 0; a < D; ++a)
            for (int b = a; b < D; ++b) {
                double s = 0;
                const double* ca = &col[(size_t)a * D];
                const double* cb = &col[(size_t)b * D];
                for (int i = 0; i < D; ++i) s += ca[i] * cb[i];
                worst = std::max(worst, std::fabs(s - (a == b ? 1.0 : 0.0)));
            }
        if (worst > 1e-4) return fail(PA_EBASIS, "basis not orthonormal: max|VtV-I| = %.3g", worst);
    }
    for (int64_t u = 0; u < n; ++u)
        if (member[u])
            for (int j = 0; j < dp; ++j)
                if (!std::isfinite(p->reduced[u * rsin + j])) return fail(PA_EINVAL, "non-finite reduced[%lld]", (long long)u);
    // ---- FES index
    const int r = p->fes_r;
    if (p->fes_cell_off[0] != 0) return fail(PA_EFES, "fes_cell_off[0] != 0");
    for (int c = 0; c < r; ++c)
        if (p->fes_cell_off[c + 1] <= p->fes_cell_off[c]) return fail(PA_EFES, "FES cell %d is empty", c);
    const int64_t pool_n = p->fes_cell_off[r];
    int64_t max_cell = 0;
    for (int c = 0; c < r; ++c) max_cell = std::max<int64_t>(max_cell, p->fes_cell_off[c + 1] - p->fes_cell_off[c]);
    if (pool_n >= (1ll << 31)) return fail(PA_EFES, "pool too large");
    {
        std::vector<uint8_t> seen(n, 0);
        for (int64_t j = 0; j < pool_n; ++j) {
            int32_t e = p->fes_pool_ids[j];
            if (e < 0 || e >= n) return fail(PA_EFES, "pool id %d out of range", e);
            if (!member[e]) return fail(PA_EFES, "pool id %d is not a member", e);
            if (seen[e]) return fail(PA_EFES, "pool id %d duplicated", e);
            seen[e] = 1;
        }
    }
    for (int64_t i = 0; i < (int64_t)r * dp; ++i)
        if (!std::isfinite(p->fes_centroids[i])) return fail(PA_EINVAL, "non-finite centroid");

    // NEXT-f1 storage: reduced rows rounded once to binary16 (RNE); every stage-①
    // distance and the FES pool then use exactly these rounded values.
    std::vector<float> red16;
    const float* RED = p->reduced;
    if (p->reduced_fp16) {
        red16.resize((size_t)n * dp);
        bool bad = false;
        parallel_rows(n, [&](int64_t lo, int64_t hi) {
            for (int64_t u = lo; u < hi; ++u)
                for (int j = 0; j < dp; ++j) {
                    const float v = __half2float(__float2half_rn(p->reduced[u * rsin + j]));
                    red16[u * dp + j] = v;
                    if (!std::isfinite(v) && member[u]) bad = true;
                }
        });
        if (bad) return fail(PA_EINVAL, "reduced value outside the binary16 range");
        RED = red16.data();
        rsin = dp;
    }
    // ---- device replica
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (p->device < 0 || p->device >= ndev) return fail(PA_EINVAL, "device %d not in [0,%d)", p->device, ndev);
    CU(cudaSetDevice(p->device));
    int major = 0, minor = 0;
    CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device));
    CU(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, p->device));
    if (major != 10 || minor != 0)
        return fail(PA_ENOTSUP, "device %d is sm_%d%d; this library is built for sm_100a only", p->device, major, minor);

    pa_index* ix = new pa_index();
    ix->device = p->device;
    auto& d = ix->dev;
    d.n = n; d.dim = D; d.rdim = dp; d.rdim_pad = (dp + 3) & ~3; d.metric = p->metric; d.fes_r = r;
    d.pool_n = pool_n;
    d.max_cell = (int32_t)((max_cell + 3) & ~3);
    d.ell_w = p->max_degree <= 32 ? 32 : 64;
    const int dps = d.rdim_pad;
    d.rdim_h = (dp + 7) & ~7;
    d.qlen = p->reduced_fp16 ? std::max(dps, d.rdim_h) : dps;
    const bool f16 = p->reduced_fp16 != 0;
    // Rows start on 128-B lines and the traversal reads each with 8 lanes × 16 B per
    // load (whole lines of 4 rows per instruction): the stride is rounded up to 128 B
    // (e.g. d' = 48 fp32: 192 B of data in a 256-B slot); the padding is never read.
    d.rstride = (dps + 31) & ~31;
    d.rstride_h = (d.rdim_h + 63) & ~63;
    const int rs = f16 ? d.rstride_h : d.rstride;
    auto bail = [&](pa_status s) { pa_destroy(ix); return s; };
    {
        std::lock_guard<std::mutex> g(g_reg_mu);
        g_live.insert(ix);
    }
#define CUB(expr)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return bail(fail(e_ == cudaErrorMemoryAllocation ? PA_ENOMEM : PA_ECUDA, "%s: %s", #expr, \
                             cudaGetErrorString(e_)));                                             \
    } while (0)
    CUB(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    CUB(cudaStreamCreateWithFlags(&ix->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ix->ev) CUB(cudaEventCreate(&e));
    CUB(cudaEventCreateWithFlags(&ix->done_ev, cudaEventDisableTiming));
    CUB(dalloc(&d.basis, (size_t)D * D));
    CUB(cudaMemcpy(d.basis, p->basis, sizeof(float) * D * D, cudaMemcpyHostToDevice));
    // reduced vectors [n][dps] fp32 or [n][rdim_h] binary16 (zero rows for non-members), staged in chunks
    if (f16) {
        __half* rh = nullptr;
        CUB(cudaMalloc((void**)&rh, sizeof(__half) * (size_t)n * d.rstride_h));
        d.reduced_h = rh;
    } else {
        CUB(dalloc(&d.reduced, (size_t)n * d.rstride));
    }
    CUB(dalloc(&d.ell, (size_t)n * d.ell_w));
    {
        const int64_t chunk = 1 << 20;
        std::vector<float> rb(f16 ? 0 : (size_t)std::min(chunk, n) * rs);
        std::vector<__half> hb(f16 ? (size_t)std::min(chunk, n) * rs : 0);
        std::vector<int32_t> eb((size_t)std::min(chunk, n) * d.ell_w);
        for (int64_t s0 = 0; s0 < n; s0 += chunk) {
            int64_t s1 = std::min(n, s0 + chunk);
            parallel_rows(s1 - s0, [&](int64_t lo, int64_t hi) {
                for (int64_t i = lo; i < hi; ++i) {
                    int64_t u = s0 + i;
                    if (f16) {
                        __half* dh = &hb[(size_t)i * rs];
                        for (int j = 0; j < rs; ++j)
                            dh[j] = __float2half_rn(member[u] && j < dp ? RED[u * rsin + j] : 0.f);
                    } else {
                        float* dst = &rb[(size_t)i * rs];
                        if (member[u]) {
                            std::memcpy(dst, RED + u * rsin, sizeof(float) * dp);
                            for (int j = dp; j < rs; ++j) dst[j] = 0.f;
                        } else {
                            std::memset(dst, 0, sizeof(float) * rs);
                        }
                    }
                    int32_t* row = &eb[(size_t)i * d.ell_w];
                    int64_t a0 = p->sub_offsets[u], a1 = p->sub_offsets[u + 1];
                    for (int j = 0; j < d.ell_w; ++j) row[j] = (a0 + j < a1) ? p->sub_neighbors[a0 + j] : -1;
                }
            });
            if (f16)
                CUB(cudaMemcpy(static_cast<__half*>(d.reduced_h) + s0 * rs, hb.data(),
                               sizeof(__half) * (s1 - s0) * rs, cudaMemcpyHostToDevice));
            else
                CUB(cudaMemcpy(d.reduced + s0 * rs, rb.data(), sizeof(float) * (s1 - s0) * rs, cudaMemcpyHostToDevice));
            CUB(cudaMemcpy(d.ell + s0 * d.ell_w, eb.data(), sizeof(int32_t) * (s1 - s0) * d.ell_w, cudaMemcpyHostToDevice));
        }
    }
    // FES: centroids, cell offsets, pool ids and pool vectors grouped by cell
    {
        std::vector<float> cb((size_t)r * dps, 0.f);
        for (int c = 0; c < r; ++c) std::memcpy(&cb[(size_t)c * dps], p->fes_centroids + (size_t)c * dp, sizeof(float) * dp);
        CUB(dalloc(&d.centroids, cb.size()));
        CUB(cudaMemcpy(d.centroids, cb.data(), sizeof(float) * cb.size(), cudaMemcpyHostToDevice));
        std::vector<int32_t> co(r + 1);
        for (int c = 0; c <= r; ++c) co[c] = (int32_t)p->fes_cell_off[c];
        CUB(dalloc(&d.cell_off, co.size()));
        CUB(cudaMemcpy(d.cell_off, co.data(), sizeof(int32_t) * co.size(), cudaMemcpyHostToDevice));
        CUB(dalloc(&d.pool_ids, (size_t)pool_n));
        CUB(cudaMemcpy(d.pool_ids, p->fes_pool_ids, sizeof(int32_t) * pool_n, cudaMemcpyHostToDevice));
        std::vector<float> pv((size_t)pool_n * dps, 0.f);
        for (int64_t j = 0; j < pool_n; ++j)
            std::memcpy(&pv[(size_t)j * dps], RED + (int64_t)p->fes_pool_ids[j] * rsin, sizeof(float) * dp);
        CUB(dalloc(&d.pool_vec, pv.size()));
        CUB(cudaMemcpy(d.pool_vec, pv.data(), sizeof(float) * pv.size(), cudaMemcpyHostToDevice));
        std::vector<float> pn((size_t)pool_n);
        for (int64_t j = 0; j < pool_n; ++j) {
            double s2 = 0;
            const float* e = RED + (int64_t)p->fes_pool_ids[j] * rsin;
            for (int i = 0; i < dp; ++i) s2 += (double)e[i] * e[i];
            pn[j] = (float)s2;
        }
        CUB(dalloc(&d.pool_norm, pn.size()));
        CUB(cudaMemcpy(d.pool_norm, pn.data(), sizeof(float) * pn.size(), cudaMemcpyHostToDevice));
        // Pre-split, pre-swizzled pool tiles for the TMA-fed tcgen05 FES GEMM:
        // per cell, per 128-entry chunk, per 32-float K chunk: hi tile then lo tile,
        // element (row, k) at the K-major SWIZZLE_128B offset used by the kernel.
        // The score epilogue is folded into the GEMM: B row = [−2e, ‖e‖²] (L2; the
        // A row carries a 1 in column dps) or [−e] (IP), so the accumulator IS the
        // GEMM-form score ‖e‖² − 2q'·e / −q'·e.
        // (L2 needs a spare K column: d' a multiple of 32 keeps ‖e‖² in the epilogue.)
        const bool l2 = p->metric == PA_L2;
        const int kch = (dps + 31) / 32;
        d.fes_fold_norm = l2 && (dps % 32) != 0;
        std::vector<int32_t> choff(r + 1, 0);
        for (int c = 0; c < r; ++c)
            choff[c + 1] = choff[c] + (int32_t)((p->fes_cell_off[c + 1] - p->fes_cell_off[c] + 127) / 128);
        std::vector<float> img((size_t)choff[r] * kch * 2 * 4096, 0.f);
        auto swz = [](int row, int k) {
            return (size_t)((row >> 3) * 256 + (row & 7) * 32 + (((k >> 2) ^ (row & 7)) << 2) + (k & 3));
        };
        for (int c = 0; c < r; ++c) {
            const int64_t b = p->fes_cell_off[c], nc = p->fes_cell_off[c + 1] - b;
            for (int64_t e = 0; e < nc; ++e) {
                const int ch = choff[c] + (int)(e / 128), row = (int)(e % 128);
                const float* src = RED + (int64_t)p->fes_pool_ids[b + e] * rsin;
                for (int kc = 0; kc < kch; ++kc) {
                    float* hi = &img[(((size_t)ch * kch + kc) * 2 + 0) * 4096];
                    float* lo = &img[(((size_t)ch * kch + kc) * 2 + 1) * 4096];
                    for (int k = 0; k < 32; ++k) {
                        const int col = kc * 32 + k;
                        const float a = col < dp ? (l2 ? -2.f * src[col] : -src[col])
                                                 : (d.fes_fold_norm && col == dps ? pn[b + e] : 0.f);
                        uint32_t bits;
                        std::memcpy(&bits, &a, 4);
                        bits &= 0xFFFFE000u;
                        float h;
                        std::memcpy(&h, &bits, 4);
                        hi[swz(row, k)] = h;
                        lo[swz(row, k)] = a - h;
                    }
                }
            }
        }
        CUB(dalloc(&d.pool_img, img.size()));
        CUB(cudaMemcpy(d.pool_img, img.data(), sizeof(float) * img.size(), cudaMemcpyHostToDevice));
        d.pool_chunks = choff[r];
        CUB(dalloc(&d.chunk_off, choff.size()));
        CUB(cudaMemcpy(d.chunk_off, choff.data(), sizeof(int32_t) * choff.size(), cudaMemcpyHostToDevice));
    }
    // tcgen05 projection operand B_T = [(V_{:d'}·Cᵀ)ᵀ ; Vᵀ] (rows K-major), fp64 → fp32, split to TF32
    // hi/lo and laid out per 32-float K chunk as two planes of [NB][32] in K-major SWIZZLE_128B order
    // (the same element placement as the FES pool tiles), zero-padded to NB = roundup16(r + D) rows.
    {
        const int NB = ((r + D) + 15) & ~15;
        const int kch = (D + 31) / 32;
        std::vector<float> bt((size_t)NB * D, 0.f);
        for (int c = 0; c < r; ++c)
            for (int k = 0; k < D; ++k) {
                double s = 0;
                for (int j = 0; j < dp; ++j) s += (double)p->basis[(size_t)k * D + j] * (double)p->fes_centroids[(size_t)c * dp + j];
                bt[(size_t)c * D + k] = (float)s;
            }
        for (int j = 0; j < D; ++j)
            for (int k = 0; k < D; ++k) bt[(size_t)(r + j) * D + k] = p->basis[(size_t)k * D + j];
        std::vector<float> img((size_t)kch * 2 * NB * 32, 0.f);
        for (int n = 0; n < NB; ++n)
            for (int k = 0; k < kch * 32; ++k) {
                const float a = k < D ? bt[(size_t)n * D + k] : 0.f;
                uint32_t bits;
                std::memcpy(&bits, &a, 4);
                bits &= 0xFFFFE000u;
                float h;
                std::memcpy(&h, &bits, 4);
                const int kc = k >> 5, kk = k & 31;
                const size_t in_row = (size_t)n * 32 + ((((kk >> 2) ^ (n & 7)) << 2) | (kk & 3));
                img[((size_t)kc * 2 + 0) * NB * 32 + in_row] = h;
                img[((size_t)kc * 2 + 1) * NB * 32 + in_row] = a - h;
            }
        std::vector<float> cn(r);
        for (int c = 0; c < r; ++c) {
            double s = 0;
            for (int j = 0; j < dp; ++j) s += (double)p->fes_centroids[(size_t)c * dp + j] * p->fes_centroids[(size_t)c * dp + j];
            cn[c] = (float)s;
        }
        d.proj_nb = NB;
        CUB(dalloc(&d.proj_img, img.size()));
        CUB(cudaMemcpy(d.proj_img, img.data(), sizeof(float) * img.size(), cudaMemcpyHostToDevice));
        CUB(dalloc(&d.cent_norm, cn.size()));
        CUB(cudaMemcpy(d.cent_norm, cn.data(), sizeof(float) * cn.size(), cudaMemcpyHostToDevice));
    }
    ix->h_sub_off.assign(p->sub_offsets, p->sub_offsets + n + 1);
    ix->h_sub_nb.assign(p->sub_neighbors, p->sub_neighbors + p->sub_offsets[n]);
    CUB(cudaDeviceSynchronize());
#undef CUB
    *out = ix;
    return PA_OK;
}

pa_status pa_attach_host(pa_index* ix, const int64_t* full_offsets, const int32_t* full_neighbors,
                         const float* rotated_full) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (!full_offsets || !full_neighbors || !rotated_full) return fail(PA_EINVAL, "null argument");
    pa_status st = check_csr(full_offsets, full_neighbors, ix->dev.n, 0, "full graph");
    if (st != PA_OK) return st;
    std::lock_guard<std::mutex> g(ix->mu);
    ix->h_full_off = full_offsets;
    ix->h_full_nb = full_neighbors;
    ix->h_rotated = rotated_full;
    return PA_OK;
}

pa_status pa_search_device(pa_index* ix, const float* d_queries, int64_t m, int32_t k, int32_t ef,
                           const pa_search_opts* opts, int32_t* d_out_ids, float* d_out_dists,
                           const pa_debug* dbg, void* stream) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (m < 0) return fail(PA_EINVAL, "m < 0");
    if (m > 0 && (!d_queries || !d_out_ids || !d_out_dists)) return fail(PA_EINVAL, "null argument");
    Resolved r;
    pa_status st = resolve(opts, k, ef, &r, ix->dev.n);
    if (st != PA_OK) return st;
    if (r.stages == PA_STAGES_FULL) return fail(PA_EINVAL, "pa_search_device runs on the GPU only (stages 1 or 7)");
    std::lock_guard<std::mutex> g(ix->mu);
    CU(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)stream;          // NULL = the legacy default stream (CUDA convention)
    if (m == 0) return PA_OK;
    if (r.stages == PA_STAGES_FULL_GPU) {
        st = ensure_full_device(ix);
        if (st != PA_OK) return st;
    }
    return enqueue_gpu_stage(ix, d_queries, m, k, r, d_out_ids, d_out_dists, dbg, r.stages == PA_STAGES_FULL_GPU, s);
}

static pa_status search_host_impl(pa_index* ix, const float* queries, int64_t m, int32_t k, const Resolved& r,
                                  int32_t* out_ids, float* out_d, bool candidates_only) {
    auto t0 = std::chrono::steady_clock::now();
    CU(cudaSetDevice(ix->device));
    cudaStream_t s = ix->stream;
    const bool full = !candidates_only && r.stages == PA_STAGES_FULL;
    if (full && (!ix->h_rotated || !ix->h_full_off))
        return fail(PA_ESTATE, "PA_STAGES_FULL requires pa_attach_host");
    if (full && ix->h_sub_off.empty())
        return fail(PA_ESTATE, "PA_STAGES_FULL: this replica has no host copy of the subgraph (built by pa_build_replica)");
    if (!candidates_only && r.stages == PA_STAGES_FULL_GPU) {
        pa_status st0 = ensure_full_device(ix);
        if (st0 != PA_OK) return st0;
    }
    pa_status st = ensure_ws(ix, m, r.E, r.ef1, k);
    if (st != PA_OK) return st;
    const auto& d = ix->dev;
    // Stages ②③ pipeline over sub-batches (GPU stage of batch j+1 overlaps host work on j).
    const int64_t bsz = full && !(r.flags & PA_NO_PIPELINE) ? std::max<int64_t>(1024, (m + 7) / 8) : m;
    const int64_t nb = (m + bsz - 1) / bsz;
    if (full) {
        st = ensure_pipe_events(ix, nb);
        if (st != PA_OK) return st;
        CU(cudaEventRecord(ix->pipe_start, s));
    }
    const int64_t m0 = std::min(m, bsz);
    CU(cudaMemcpyAsync(ix->q, queries, sizeof(float) * m0 * d.dim, cudaMemcpyHostToDevice, s));
    st = enqueue_gpu_stage(ix, ix->q, m0, k, r, ix->out_ids, ix->out_d, nullptr,
                           full || r.stages == PA_STAGES_FULL_GPU, s);
    if (st != PA_OK) return st;
    int64_t launches = ix->stats.kernel_launches;
    if (candidates_only) {
        CU(cudaMemcpyAsync(out_ids, ix->cand_ids, sizeof(int32_t) * m * r.ef1, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(out_d, ix->cand_d, sizeof(float) * m * r.ef1, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    } else if (!full) {
        CU(cudaMemcpyAsync(out_ids, ix->out_ids, sizeof(int32_t) * m * k, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(out_d, ix->out_d, sizeof(float) * m * k, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    } else {
        st = ensure_host_ws(ix, m, r.ef1);
        if (st != PA_OK) return st;
        // The first sub-batch was enqueued above; the rest are enqueued now so the
        // GPU stage of batch j+1.. runs while the host refines batch j (A12).
        std::vector<int64_t> lo(nb + 1);
        for (int64_t j = 0; j <= nb; ++j) lo[j] = std::min<int64_t>(m, j * bsz);
        for (int64_t j = 0; j < nb; ++j) {
            const int64_t a0 = lo[j], mj = lo[j + 1] - lo[j];
            if (j > 0) {
                CU(cudaMemcpyAsync(ix->q + a0 * d.dim, queries + a0 * d.dim, sizeof(float) * mj * d.dim,
                                   cudaMemcpyHostToDevice, s));
                st = enqueue_gpu_stage(ix, ix->q + a0 * d.dim, mj, k, r, ix->out_ids + a0 * k, ix->out_d + a0 * k,
                                       nullptr, true, s, a0);
                if (st != PA_OK) return st;
                launches += ix->stats.kernel_launches;
            }
            CU(cudaEventRecord(ix->pipe_done[j], s));
            CU(cudaStreamWaitEvent(ix->copy_stream, ix->pipe_done[j], 0));
            cudaStream_t c = ix->copy_stream;
            CU(cudaMemcpyAsync(ix->h_cand_ids + a0 * r.ef1, ix->cand_ids + a0 * r.ef1, sizeof(int32_t) * mj * r.ef1,
                               cudaMemcpyDeviceToHost, c));
            CU(cudaMemcpyAsync(ix->h_cand_d + a0 * r.ef1, ix->cand_d + a0 * r.ef1, sizeof(float) * mj * r.ef1,
                               cudaMemcpyDeviceToHost, c));
            CU(cudaMemcpyAsync(ix->h_qp + a0 * d.rdim_pad, ix->qp + a0 * d.rdim_pad, sizeof(float) * mj * d.rdim_pad,
                               cudaMemcpyDeviceToHost, c));
            if (d.dim > d.rdim)
                CU(cudaMemcpyAsync(ix->h_qres + a0 * (d.dim - d.rdim), ix->qres + a0 * (d.dim - d.rdim),
                                   sizeof(float) * mj * (d.dim - d.rdim), cudaMemcpyDeviceToHost, c));
            CU(cudaEventRecord(ix->pipe_copied[j], c));
        }
        CU(cudaEventRecord(ix->pipe_end, s));
        // One pass of the host worker pool over all m queries; a worker entering a
        // new sub-batch waits for that sub-batch's D2H event only.
        struct Ready {
            pa_index* ix;
            int64_t bsz;
            std::vector<std::atomic<int>> done;
            explicit Ready(size_t n) : done(n) {}
        } ready(nb);
        ready.ix = ix;
        ready.bsz = bsz;
        for (auto& x : ready.done) x.store(0);
        auto th = std::chrono::steady_clock::now();
        pa::HostStageArgs h;
        h.dim = d.dim; h.rdim = d.rdim; h.metric = d.metric;
        h.sub.off = ix->h_sub_off.data(); h.sub.nb = ix->h_sub_nb.data();
        h.full.off = ix->h_full_off; h.full.nb = ix->h_full_nb;
        h.rotated = ix->h_rotated;
        h.m = m; h.k = k; h.ef1 = r.ef1; h.ef2 = r.ef2; h.ef3 = r.ef3; h.refine_iters = r.refine; h.width = r.width;
        h.flags = r.flags; h.threads = r.threads;
        h.cand_ids = ix->h_cand_ids; h.cand_d = ix->h_cand_d; h.qp = ix->h_qp; h.qp_stride = d.rdim_pad;
        h.qres = ix->h_qres; h.out_ids = out_ids; h.out_d = out_d;
        h.recompute_primary = d.reduced_h != nullptr;   // δ' was computed on rounded rows
        int64_t s2 = 0, s3 = 0;
        h.sum_n_dist2 = &s2; h.sum_n_dist3 = &s3;
        h.ready_ctx = &ready;
        h.wait_ready = [](void* ctx, int64_t q) {
            Ready* R = static_cast<Ready*>(ctx);
            const int64_t j = q / R->bsz;
            if (R->done[j].load(std::memory_order_acquire)) return;
            cudaEventSynchronize(R->ix->pipe_copied[j]);
            R->done[j].store(1, std::memory_order_release);
        };
        pa::run_host_stages(h);
        const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th).count();
        CU(cudaStreamSynchronize(s));
        float gpu_ms = 0;
        cudaEventElapsedTime(&gpu_ms, ix->pipe_start, ix->pipe_end);
        ix->stats = pa_stats{};
        ix->stats.queries = m;
        ix->stats.ms_total_gpu = gpu_ms;
        ix->stats.ms_host_stages = host_ms;
        ix->stats.sum_n_dist2 = s2; ix->stats.sum_n_dist3 = s3;
        ix->events_pending = false;
    }
    collect_event_times(ix);
    ix->stats.kernel_launches = launches;
    ix->stats.ms_wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return PA_OK;
}

pa_status pa_search(pa_index* ix, const float* queries, int64_t m, int32_t k, int32_t ef,
                    const pa_search_opts* opts, int32_t* out_ids, float* out_dists) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (m < 0) return fail(PA_EINVAL, "m < 0");
    if (m > 0 && (!queries || !out_ids || !out_dists)) return fail(PA_EINVAL, "null argument");
    Resolved r;
    pa_status st = resolve(opts, k, ef, &r, ix->dev.n);
    if (st != PA_OK) return st;
    std::lock_guard<std::mutex> g(ix->mu);
    if (m == 0) return PA_OK;
    return search_host_impl(ix, queries, m, k, r, out_ids, out_dists, false);
}

pa_status pa_search_candidates(pa_index* ix, const float* queries, int64_t m, int32_t ef,
                               const pa_search_opts* opts, int32_t* cand_ids, float* cand_dists) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (m < 0) return fail(PA_EINVAL, "m < 0");
    if (m > 0 && (!queries || !cand_ids || !cand_dists)) return fail(PA_EINVAL, "null argument");
    Resolved r;
    pa_status st = resolve(opts, 1, ef, &r, ix->dev.n);
    if (st != PA_OK) return st;
    if (opts && opts->ef1 && opts->ef1 != ef) return fail(PA_EINVAL, "candidates are [m][ef]: ef1 must equal ef");
    if (r.stages != PA_STAGES_GPU)
        return fail(PA_EINVAL, "pa_search_candidates returns stage-1 lists: stages must be 0 or PA_STAGES_GPU");
    std::lock_guard<std::mutex> g(ix->mu);
    if (m == 0) return PA_OK;
    return search_host_impl(ix, queries, m, 1, r, cand_ids, cand_dists, true);
}

pa_status pa_entries_device(pa_index* ix, const float* d_queries, int64_t m, int32_t E, int32_t method,
                            int32_t e0, int32_t beam, int32_t* d_entries, float* d_entry_dists,
                            int32_t* d_n_dist, void* stream) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (m < 0) return fail(PA_EINVAL, "m < 0");
    if (E < 1 || E > 256) return fail(PA_EINVAL, "E = %d (1..256)", E);
    if (method != PA_ENTRIES_FES && method != PA_ENTRIES_TWO_HOP) return fail(PA_EINVAL, "unknown method %d", method);
    if (method == PA_ENTRIES_TWO_HOP) {
        if (beam < 0) return fail(PA_EINVAL, "beam < 0");
        if (e0 < 0 || (int64_t)e0 >= ix->dev.n) return fail(PA_EINVAL, "e0 = %d outside [0, n)", e0);
        if (!pa::two_hop_supported(ix->dev, E))
            return fail(PA_ENOTSUP, "two-hop entries need an ELL-32, fp32-row index");
    }
    if (m > 0 && (!d_queries || !d_entries)) return fail(PA_EINVAL, "null argument");
    std::lock_guard<std::mutex> g(ix->mu);
    CU(cudaSetDevice(ix->device));
    if (m == 0) return PA_OK;
    pa_status st = ensure_ws(ix, m, E, E, 1);
    if (st != PA_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (ix->done_recorded) CU(cudaStreamWaitEvent(s, ix->done_ev, 0));
    pa::SearchArgs a;
    a.m = m; a.k = 1; a.ef = E; a.E = E;
    a.q = d_queries; a.qp = ix->qp; a.qres = nullptr; a.cell = ix->cell; a.entries = d_entries;
    a.perm = ix->perm; a.qoff = ix->qoff; a.toff = ix->toff; a.fes_scores = ix->fes_scores;
    a.work = ix->work;
    int launches = 0;
    CU(cudaEventRecord(ix->ev[0], s));
    if (pa::project_tc_supported(ix->dev, false)) {
        launches += pa::launch_project_tc(ix->dev, a, s);
        a.cell_ready = true;
    } else {
        launches += pa::launch_project(ix->dev, a, s);
    }
    CU(cudaGetLastError());
    CU(cudaEventRecord(ix->ev[1], s));
    if (method == PA_ENTRIES_FES) {
        if (a.cell_ready && pa::fes_tc_supported(ix->dev, E)) launches += pa::launch_fes_tc(ix->dev, a, s);
        else launches += pa::launch_fes(ix->dev, a, s);
    } else {
        pa::TwoHopArgs t;
        t.m = m; t.E = E; t.beam = beam; t.e0 = e0; t.qp = ix->qp;
        t.entries = d_entries; t.entry_d = d_entry_dists; t.n_dist = d_n_dist;
        launches += pa::launch_two_hop(ix->dev, t, s);
    }
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(ix->counters, 0, sizeof(int32_t) * 4 * (size_t)m, s));   // no stage-① counters
    for (int i = 2; i < 5; ++i) CU(cudaEventRecord(ix->ev[i], s));
    CU(cudaEventRecord(ix->done_ev, s));
    ix->done_recorded = true;
    ix->events_pending = true;
    ix->last_full_gpu = false;
    ix->stats = pa_stats{};
    ix->stats.queries = m;
    ix->stats.kernel_launches = launches;
    return PA_OK;
}

pa_status pa_replica_meta_of(const pa_index* ix, pa_replica_meta* out) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (!out) return fail(PA_EINVAL, "null argument");
    const auto& d = ix->dev;
    pa_replica_meta m{};
    m.n = d.n; m.pool_n = d.pool_n; m.dim = d.dim; m.rdim = d.rdim; m.rdim_pad = d.rdim_pad; m.rdim_h = d.rdim_h;
    m.qlen = d.qlen; m.rstride = d.rstride; m.rstride_h = d.rstride_h; m.ell_w = d.ell_w; m.metric = d.metric;
    m.fes_r = d.fes_r; m.max_cell = d.max_cell; m.proj_nb = d.proj_nb; m.pool_chunks = d.pool_chunks;
    m.fes_fold_norm = d.fes_fold_norm ? 1 : 0; m.reduced_fp16 = d.reduced_h ? 1 : 0;
    m.has_full = d.xhat ? 1 : 0; m.full_w = d.full_w; m.xstride = d.xstride;
    *out = m;
    return PA_OK;
}

pa_status pa_build_replica(const pa_replica_meta* m, int32_t device, pa_index** out) {
    g_err.clear();
    if (!m || !out) return fail(PA_EINVAL, "null argument");
    *out = nullptr;
    const bool ok = m->n > 0 && m->n < (1ll << 31) && m->dim > 0 && m->dim <= 4096 && m->rdim > 0 &&
                    m->rdim <= m->dim && m->rdim_pad == ((m->rdim + 3) & ~3) && m->rstride == ((m->rdim_pad + 31) & ~31) &&
                    (m->ell_w == 32 || m->ell_w == 64) && (m->metric == PA_L2 || m->metric == PA_IP) &&
                    m->fes_r >= 1 && m->fes_r <= 1024 && m->pool_n >= m->fes_r && m->pool_chunks >= m->fes_r &&
                    m->proj_nb == ((m->fes_r + m->dim + 15) & ~15) && m->max_cell > 0 &&
                    (!m->has_full || ((m->full_w == 32 || m->full_w == 64) && m->xstride == ((m->dim + 31) & ~31)));
    if (!ok) return fail(PA_EINVAL, "inconsistent replica meta");
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(PA_EINVAL, "device %d not in [0,%d)", device, ndev);
    CU(cudaSetDevice(device));
    pa_index* ix = new pa_index();
    ix->device = device;
    auto& d = ix->dev;
    d.n = m->n; d.pool_n = m->pool_n; d.dim = m->dim; d.rdim = m->rdim; d.rdim_pad = m->rdim_pad; d.rdim_h = m->rdim_h;
    d.qlen = m->qlen; d.rstride = m->rstride; d.rstride_h = m->rstride_h; d.ell_w = m->ell_w; d.metric = m->metric;
    d.fes_r = m->fes_r; d.max_cell = m->max_cell; d.proj_nb = m->proj_nb; d.pool_chunks = m->pool_chunks;
    d.fes_fold_norm = m->fes_fold_norm != 0; d.full_w = m->has_full ? m->full_w : 0; d.xstride = m->has_full ? m->xstride : 0;
    {
        std::lock_guard<std::mutex> g(g_reg_mu);
        g_live.insert(ix);
    }
    auto bail = [&](pa_status s) { pa_destroy(ix); return s; };
    // sentinel non-null pointers select the optional arrays in replica_list, then real allocations
    if (m->reduced_fp16) d.reduced_h = reinterpret_cast<void*>(1);
    if (m->has_full) d.xhat = reinterpret_cast<float*>(1);
    std::vector<std::pair<void**, size_t>> L;
    replica_list(d, L);
    for (auto& e : L) *e.first = nullptr;
    for (auto& e : L) {
        cudaError_t er = cudaMalloc(e.first, std::max<size_t>(1, e.second));
        if (er != cudaSuccess) {
            *e.first = nullptr;
            return bail(fail(er == cudaErrorMemoryAllocation ? PA_ENOMEM : PA_ECUDA, "replica allocation: %s",
                             cudaGetErrorString(er)));
        }
    }
    if (cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ix->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ix->done_ev, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(PA_ECUDA, "replica streams"));
    for (auto& e : ix->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(PA_ECUDA, "replica events"));
    *out = ix;
    return PA_OK;
}

pa_status pa_replica_buffers(pa_index* ix, pa_buffer* out, int32_t cap, int32_t* count) {
    g_err.clear();
    if (!live(ix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (!count || (cap > 0 && !out)) return fail(PA_EINVAL, "null argument");
    std::lock_guard<std::mutex> g(ix->mu);
    std::vector<std::pair<void**, size_t>> L;
    replica_list(ix->dev, L);
    for (int32_t i = 0; i < cap && i < (int32_t)L.size(); ++i) {
        out[i].ptr = *L[i].first;
        out[i].bytes = (int64_t)L[i].second;
    }
    *count = (int32_t)L.size();
    return PA_OK;
}

pa_status pa_get_stats(const pa_index* cix, pa_stats* out, size_t size) {
    g_err.clear();
    if (!live(cix)) return fail(PA_ESTATE, "invalid or destroyed index handle");
    if (!out || size < sizeof(pa_stats)) return fail(PA_EINVAL, "bad stats buffer");
    pa_index* ix = const_cast<pa_index*>(cix);
    std::lock_guard<std::mutex> g(ix->mu);
    cudaSetDevice(ix->device);
    collect_event_times(ix);
    // reduce stage-① counters of the last search
    if (ix->stats.queries > 0 && ix->counters) {
        std::vector<int32_t> c((size_t)ix->stats.queries * 4);
        if (cudaMemcpy(c.data(), ix->counters, sizeof(int32_t) * c.size(), cudaMemcpyDeviceToHost) == cudaSuccess) {
            int64_t se = 0, sd = 0, ss = 0, ov = 0;
            for (int64_t q = 0; q < ix->stats.queries; ++q) {
                se += c[q * 4]; sd += c[q * 4 + 1]; ss += c[q * 4 + 2]; ov += c[q * 4 + 3] != 0;
            }
            ix->stats.sum_n_exp = se; ix->stats.sum_n_dist = sd; ix->stats.sum_spill = ss; ix->stats.overflow_queries = ov;
        }
        if (ix->last_full_gpu && ix->counters2 &&
            cudaMemcpy(c.data(), ix->counters2, sizeof(int32_t) * c.size(), cudaMemcpyDeviceToHost) == cudaSuccess) {
            int64_t s2 = 0, s3 = 0, ov = 0;
            for (int64_t q = 0; q < ix->stats.queries; ++q) {
                s2 += c[q * 4]; s3 += c[q * 4 + 1]; ov += c[q * 4 + 3] != 0;
            }
            ix->stats.sum_n_dist2 = s2; ix->stats.sum_n_dist3 = s3; ix->stats.overflow_queries += ov;
        }
    }
    std::memcpy(out, &ix->stats, sizeof(pa_stats));
    return PA_OK;
}

void pa_destroy(pa_index* ix) {
    {
        std::lock_guard<std::mutex> g(g_reg_mu);
        if (!ix || !g_live.count(ix)) return;
        g_live.erase(ix);
    }
    cudaSetDevice(ix->device);
    if (ix->stream) cudaStreamSynchronize(ix->stream);
    if (ix->copy_stream) cudaStreamSynchronize(ix->copy_stream);
    free_ws(ix);
    cudaFree(ix->spill);
    cudaFreeHost(ix->h_cand_ids); cudaFreeHost(ix->h_cand_d); cudaFreeHost(ix->h_qp); cudaFreeHost(ix->h_qres);
    cudaFreeHost(ix->h_counters);
    auto& d = ix->dev;
    cudaFree(d.basis); cudaFree(d.reduced); cudaFree(d.reduced_h); cudaFree(d.ell); cudaFree(d.centroids); cudaFree(d.cell_off);
    cudaFree(d.pool_ids); cudaFree(d.pool_vec); cudaFree(d.proj_img); cudaFree(d.cent_norm); cudaFree(d.pool_norm);
    cudaFree(d.pool_img); cudaFree(d.chunk_off); cudaFree(d.full_ell); cudaFree(d.xhat);
    for (auto& e : ix->ev) if (e) cudaEventDestroy(e);
    if (ix->done_ev) cudaEventDestroy(ix->done_ev);
    for (auto e : ix->pipe_done) cudaEventDestroy(e);
    for (auto e : ix->pipe_copied) cudaEventDestroy(e);
    if (ix->pipe_start) cudaEventDestroy(ix->pipe_start);
    if (ix->pipe_end) cudaEventDestroy(ix->pipe_end);
    if (ix->stream) cudaStreamDestroy(ix->stream);
    if (ix->copy_stream) cudaStreamDestroy(ix->copy_stream);
    ix->magic = 0;
    delete ix;
}

}  // extern "C"
