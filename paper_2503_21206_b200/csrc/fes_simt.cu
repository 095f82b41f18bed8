// a2 + a4 — Fast Entry Selection, SIMT first cut (warp per query).
//   routing : cell(q) = argmin_c δ(q', centroid_c), ties → lower c   (Q9)
//   scoring : δ(q', e) for every pool entry e of the routed cell; keep the E
//             smallest (δ, id) keys                                  (Alg 2; Q8, Q10)
// The tensor-core version (fes_tc.cu) computes the same selection from a
// tcgen05 grouped GEMM; this kernel is kept for small batches and as the
// reference point of the tcgen05 path in tests.
#include "common.cuh"
#include "internal.h"

namespace pa {

namespace {
constexpr int kWarps = 4;

template <int METRIC, int SMAX>
__global__ void __launch_bounds__(kWarps * 32) k_fes_simt(DevIndex ix, SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int dps = ix.rdim_pad, E = a.E;
    // per-warp smem: q'[dps] | C[E]   (16-B aligned slices)
    const size_t per_warp = ((size_t)dps * 4 + (size_t)E * 8 + 15) & ~(size_t)15;
    unsigned char* base = smem_raw + per_warp * w;
    float* qs = reinterpret_cast<float*>(base);
    uint64_t* C = reinterpret_cast<uint64_t*>(base + (size_t)dps * 4);
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t q = (int64_t)blockIdx.x * kWarps + w; q < a.m; q += nwarps) {
        for (int i = lane; i < dps; i += 32) qs[i] = a.qp[q * dps + i];
        __syncwarp();
        // ---- routing (a2): direct form here unless the tcgen05 projection already routed
        int cell;
        if (a.cell_ready) {
            cell = a.cell[q];
        } else {
            uint64_t best = kKeyInf;
            for (int c = lane; c < ix.fes_r; c += 32) {
                float d = row_dist<METRIC>(qs, ix.centroids + (int64_t)c * dps, dps);
                uint64_t key = ((uint64_t)ord_of(d) << 32) | (uint32_t)c;
                best = key < best ? key : best;
            }
            best = warp_min64(best);
            cell = (int)(uint32_t)best;
            if (lane == 0 && a.cell) a.cell[q] = cell;
        }
        int32_t* out = a.entries + q * E;
        if (a.flags & 1u) {                             // PA_NO_FES: first E pool ids in pool order
            for (int j = lane; j < E; j += 32) out[j] = j < ix.pool_n ? ix.pool_ids[j] : -1;
            __syncwarp();
            continue;
        }
        // ---- within-cell scoring + top-E (a4)
        const int b = ix.cell_off[cell], e = ix.cell_off[cell + 1];
        int csz = 0;
        for (int j0 = b; j0 < e; j0 += 32) {
            const int j = j0 + lane;
            uint64_t key = kKeyInf;
            if (j < e) key = make_key(row_dist<METRIC>(qs, ix.pool_vec + (int64_t)j * dps, dps), ix.pool_ids[j]);
            const uint64_t thresh = csz == E ? C[E - 1] : kKeyInf;
            const bool pass = key < thresh;
            const unsigned pb = __ballot_sync(kFull, pass);
            if (pb == 0) continue;
            int minr;
            csz = rank_merge<SMAX>(C, csz, E, key, pass, pb, lane, minr);
        }
        for (int j = lane; j < E; j += 32) out[j] = j < csz ? key_id(C[j]) : -1;
        __syncwarp();
    }
}
}  // namespace

int launch_fes(const DevIndex& ix, const SearchArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    const size_t per_warp = ((size_t)ix.rdim_pad * 4 + (size_t)a.E * 8 + 15) & ~(size_t)15;
    const size_t smem = per_warp * kWarps;
    int64_t blocks = (a.m + kWarps - 1) / kWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    void* fn;
    const int smax = (a.E + 31) / 32;
    if (ix.metric == 0)
        fn = smax <= 2 ? (void*)k_fes_simt<0, 2> : smax <= 4 ? (void*)k_fes_simt<0, 4> : smax <= 8 ? (void*)k_fes_simt<0, 8>
                                                                                        : (void*)k_fes_simt<0, 32>;
    else
        fn = smax <= 2 ? (void*)k_fes_simt<1, 2> : smax <= 4 ? (void*)k_fes_simt<1, 4> : smax <= 8 ? (void*)k_fes_simt<1, 8>
                                                                                        : (void*)k_fes_simt<1, 32>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    DevIndex ii = ix;
    SearchArgs aa = a;
    void* args[] = {&ii, &aa};
    cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(kWarps * 32), args, smem, s);
    return 1;
}

}  // namespace pa
