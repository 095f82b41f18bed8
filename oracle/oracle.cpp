// ============================================================================
// oracle/oracle.cpp — PilotANN (arXiv 2503.21206) reference ORACLE.
//
// TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU implementation
// of what the GPU stage (and the host stages ②③) compute, in fp64, written
// step by step in the paper's order and notation.  Only tests/, the
// __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
// arms may load this library.  It shares no code, header, table or helper with
// the product library (paper_2503_21206_b200/csrc); every struct below is
// declared here and mirrored by hand in oracle/__init__.py.
//
// Citations: P:Lnnn = /root/reference/PAPER.md line, S:Lnnn = SPEC.md line.
// Readings of silent/ambiguous passages are SURVEY.md §8.c Q1–Q28, listed in
// DESIGN.md §"Readings".
//
//   O1  projection            q̂ = q·V (fp64), q' = q̂[0:d'], q_res = q̂[d':D]   P:L244-245 (§4.1 ①); Q2, Q3
//   O2  distance              L2: Σ(a_i−b_i)²  (squared, no sqrt)
//                             IP: −Σ a_i b_i   (Q1); keys ordered by (δ, id)  Q13
//   O3  routing               c* = argmin_c δ(q', centroid_c), tie → smaller c  P:L440, P:L458 (Alg 2 l.8); Q9
//   O4  FES scoring           δ'(e) for e in pool(c*); entries = min(E, n_c) smallest keys  P:L436-489 (Alg 2); Q7, Q8, Q10
//   O5  stage ① init          C := entries (≤ ef1 smallest), Vis := entries      P:L183 (Alg 1 l.3); Q15
//   O6  stage ① loop          Alg 1 lines 4-12
//   O7  stage ① output        cand1 := C                                           P:L262; Q19
//   O8  stage ② refinement    full δ re-rank, ef2, `refine_iters` expansions       P:L248-252; Q22
//   O9  stage ③ final         Alg 1 on the full graph, seeded by the carry         P:L254-258; Q23
//   O10 toggles               no-FES / no-stage1 / no-stage2
//   O11 brute force           exact top-k by (δ, id) over an id set
//   O12 recall@k              |ret_k ∩ gt_k| / k  (+ tie-aware variant)            P:L657; Q25
//   O13 bloom visited (opt.)  stage-① visited set as a partitioned bloom filter   P:L392-395 (§4.3)
//                             (3 segments × 2^s bits, segment j hashes v to
//                             ((uint32)v · A_j mod 2^32) >> (32 − s)); a neighbour
//                             is "visited" iff its 3 bits are set, else its bits
//                             are set (test-then-set, in stored order).  Entries
//                             enter C unconditionally and set their bits.  Stages
//                             ②③ keep EXACT sets.  DESIGN.md reading Q17b.
//
// Parity status: every function here is pinned by tests/test_oracle.py (see its
// module docstring for the pin of each O-step).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

// ---------------------------------------------------------------- inputs ----
struct OrcIndex {
    int64_t n;                      // nodes (full id space)
    int32_t dim, rdim;              // D, d'
    int32_t metric;                 // 0 = L2 (squared), 1 = IP (δ = −dot)
    const int64_t* sub_offsets;     // [n+1]   sampled subgraph (modified CSR)
    const int32_t* sub_neighbors;   // [sub_offsets[n]]
    const float* reduced;           // [n][rdim]  x_primary
    const float* basis;             // [dim][dim] V, columns by descending σ
    int32_t fes_r;                  // r
    const float* fes_centroids;     // [r][rdim]
    const int64_t* fes_cell_off;    // [r+1]
    const int32_t* fes_pool_ids;    // [cell_off[r]]
    const int64_t* full_offsets;    // [n+1]   full graph (stage ③); may be null
    const int32_t* full_neighbors;
    const float* rotated;           // [n][dim] X̂ = X·V (stages ②③); may be null
    int64_t reduced_stride;         // floats between rows of `reduced` (0 ⇒ rdim; dim when it is X̂ itself)
};

struct OrcOpts {
    int32_t k, ef1, ef2, ef3, entries, width, refine_iters;
    int32_t stages;                 // 1 = stage ① only, 3 = stages ①②③
    uint32_t flags;                 // 1 = no FES, 2 = no stage ②, 4 = no stage ①  (O10)
    int32_t threads;                // 0 = hardware_concurrency
    int32_t trace_cap;              // per-query capacity of stage-① traces (0 = none)
    int32_t bloom_log2;             // O13: 0 = exact stage-① visited set; s ≥ 0 bits per segment = 2^s
    int32_t use_bloom;              // 1 = O13 bloom filter in stage ① (bloom_log2 = s, may be 0)
};

struct OrcOut {
    int32_t* out_ids;  double* out_d;       // [m][k]
    int32_t* cell;                          // [m]
    int32_t* entries;  double* entries_d;   // [m][opts.entries]   (−1, +inf padded)
    int32_t* cand1_ids; double* cand1_d;    // [m][ef1]            (−1, +inf padded)
    int64_t* counters;                      // [m][8] see kCounter*
    int32_t* trace_expand;                  // [m][trace_cap] stage-① expansion sequence
    int32_t* trace_visit;                   // [m][trace_cap] stage-① visit sequence
    int32_t* trace_nexp;                    // [m] full lengths (may exceed trace_cap)
    int32_t* trace_nvis;                    // [m]
};

enum { kNExp1 = 0, kNDist1, kNExp2, kNDist2, kNExp3, kNDist3, kFesWork, kNumCounters = 8 };

// ------------------------------------------------------------ O2 distance ----
// δ between an fp64 query prefix and an fp32 row, summed in index order.
double delta(const double* q, const float* x, int32_t d, int32_t metric) {
    double s = 0.0;
    if (metric == 0) {
        for (int32_t i = 0; i < d; ++i) {
            double t = q[i] - (double)x[i];
            s += t * t;
        }
        return s;
    }
    for (int32_t i = 0; i < d; ++i) s += q[i] * (double)x[i];
    return -s;
}

// A member of the candidate list C: key (δ, id) + checked flag.
struct Cand {
    double d;
    int32_t id;
    bool checked;
};
bool key_less(const Cand& a, const Cand& b) {       // Q13: ties → smaller id
    return a.d < b.d || (a.d == b.d && a.id < b.id);
}

struct Trace {
    std::vector<int32_t> expand, visit;
};

// Visited set of Alg 1 (l.6-7): exact (std::unordered_set) or, for stage ① on
// request, the O13 partitioned bloom filter.  insert(v) returns true iff v was
// not (believed) visited, and marks it visited.
struct VisitedSet {
    bool bloom = false;
    int32_t s = 0;                                   // bits per segment = 2^s
    std::unordered_set<int32_t> exact;
    std::vector<uint8_t> bits[3];                    // one byte per bit: plain, not fast
    static uint32_t bloom_bit(int32_t v, int j, int32_t s) {
        static const uint32_t A[3] = {0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du};
        uint32_t h = (uint32_t)v * A[j];             // mod 2^32
        return s == 0 ? 0u : (h >> (32 - s));
    }
    void make_bloom(int32_t s_) {
        bloom = true;
        s = s_;
        for (auto& b : bits) b.assign((size_t)1 << s, 0);
    }
    bool test(int32_t v) const {                     // all 3 bits set?
        for (int j = 0; j < 3; ++j)
            if (!bits[j][bloom_bit(v, j, s)]) return false;
        return true;
    }
    void set(int32_t v) {
        for (int j = 0; j < 3; ++j) bits[j][bloom_bit(v, j, s)] = 1;
    }
    bool insert(int32_t v) {
        if (!bloom) return exact.insert(v).second;
        if (test(v)) return false;                   // visited, or a false positive (§4.3)
        set(v);
        return true;
    }
};

// ------------------------------------------------------ O6 Alg 1
// Runs at most `max_iters` outer iterations (−1 = until no unchecked node).
// Alg 1: u ← first unchecked node in C (l.5); for unvisited v ∈ N(u) (l.6):
// mark visited (l.7), d ← δ(q, v) (l.8), C.insert (l.9); C.resize(ef) (l.11).
// Generalised to width w: the w smallest unchecked entries are expanded, their
// rows concatenated in key order (w = 1 is Alg 1 exactly).
template <class DistFn>
void greedy(const int64_t* off, const int32_t* nb, DistFn dist, int32_t ef, int32_t w,
            long max_iters, std::vector<Cand>& C, VisitedSet& vis,
            int64_t& n_exp, int64_t& n_dist, Trace* tr) {
    long it = 0;
    while (max_iters < 0 || it < max_iters) {
        std::vector<int32_t> us;                          // l.5 (C is kept sorted)
        for (Cand& c : C) {
            if (!c.checked) {
                c.checked = true;
                us.push_back(c.id);
                if ((int32_t)us.size() == w) break;
            }
        }
        if (us.empty()) break;                            // l.12: no unchecked node
        ++it;
        std::vector<Cand> fresh;
        for (int32_t u : us) {
            ++n_exp;
            if (tr) tr->expand.push_back(u);
            for (int64_t e = off[u]; e < off[u + 1]; ++e) {   // l.6, stored order
                int32_t v = nb[e];
                if (vis.insert(v)) {                           // l.7 (unvisited → visited)
                    fresh.push_back(Cand{dist(v), v, false});  // l.8
                    ++n_dist;
                    if (tr) tr->visit.push_back(v);
                }
            }
        }
        C.insert(C.end(), fresh.begin(), fresh.end());         // l.9
        std::sort(C.begin(), C.end(), key_less);
        if ((int32_t)C.size() > ef) C.resize(ef);              // l.11 (evicted stay visited, Q14)
    }
}

void search_one(const OrcIndex& ix, const float* q, const OrcOpts& o, const OrcOut& out, int64_t qi) {
    const int32_t D = ix.dim, dp = ix.rdim, metric = ix.metric;
    int64_t* cnt = out.counters ? out.counters + qi * kNumCounters : nullptr;
    int64_t local[kNumCounters] = {0};

    // ---- O1 projection: q̂ = q·V in fp64 (Q2: out-of-sample = V columns)
    std::vector<double> qh(D, 0.0);
    for (int32_t j = 0; j < D; ++j) {
        double s = 0.0;
        for (int32_t i = 0; i < D; ++i) s += (double)q[i] * (double)ix.basis[(int64_t)i * D + j];
        qh[j] = s;
    }
    const double* qp = qh.data();                          // q' = q̂[0:d']
    const int64_t rs = ix.reduced_stride ? ix.reduced_stride : dp;
    auto dprime = [&](int32_t v) { return delta(qp, ix.reduced + (int64_t)v * rs, dp, metric); };
    auto dfull = [&](int32_t v) { return delta(qh.data(), ix.rotated + (int64_t)v * D, D, metric); };

    // ---- O3 routing (Alg 2 l.8 "Q[i] not closest to block")
    int32_t cstar = 0;
    double best = std::numeric_limits<double>::infinity();
    for (int32_t c = 0; c < ix.fes_r; ++c) {
        double dc = delta(qp, ix.fes_centroids + (int64_t)c * dp, dp, metric);
        if (dc < best) { best = dc; cstar = c; }            // strict < : tie → smaller c (Q9)
    }
    if (out.cell) out.cell[qi] = cstar;

    // ---- O4 FES scoring within the routed cell (Alg 2) / O10 no-FES
    std::vector<Cand> ent;
    const int32_t E = o.entries;
    if (o.flags & 1u) {
        int64_t npool = ix.fes_cell_off[ix.fes_r];
        for (int64_t p = 0; p < npool && (int32_t)ent.size() < E; ++p) {
            int32_t e = ix.fes_pool_ids[p];
            ent.push_back(Cand{dprime(e), e, false});
        }
        std::sort(ent.begin(), ent.end(), key_less);
    } else {
        for (int64_t p = ix.fes_cell_off[cstar]; p < ix.fes_cell_off[cstar + 1]; ++p) {
            int32_t e = ix.fes_pool_ids[p];
            ent.push_back(Cand{dprime(e), e, false});
            ++local[kFesWork];                                 // Table 3: n/r per query
        }
        std::sort(ent.begin(), ent.end(), key_less);
        if ((int32_t)ent.size() > E) ent.resize(E);            // Q8: E entries (or whole cell)
    }
    if (out.entries) {
        for (int32_t j = 0; j < E; ++j) {
            bool ok = j < (int32_t)ent.size();
            out.entries[qi * E + j] = ok ? ent[j].id : -1;
            out.entries_d[qi * E + j] = ok ? ent[j].d : std::numeric_limits<double>::infinity();
        }
    }

    // ---- O5 stage ① init: C := entries, Vis := entries, n_dist := |entries| (Q15)
    Trace tr;
    Trace* trp = o.trace_cap > 0 ? &tr : nullptr;
    std::vector<Cand> C = ent;
    VisitedSet vis;
    if (o.use_bloom) vis.make_bloom(o.bloom_log2);    // O13 (stage ① only)
    for (const Cand& c : ent) {
        if (vis.bloom) vis.set(c.id);                  // entries enter C unconditionally (O13)
        else vis.insert(c.id);
        if (trp) trp->visit.push_back(c.id);
    }
    local[kNDist1] = (int64_t)ent.size();
    if ((int32_t)C.size() > o.ef1) C.resize(o.ef1);           // resize(ef) semantics

    // ---- O6 stage ① loop on the subgraph with reduced δ'
    if (!(o.flags & 4u))
        greedy(ix.sub_offsets, ix.sub_neighbors, dprime, o.ef1, o.width, -1, C, vis,
               local[kNExp1], local[kNDist1], trp);

    // ---- O7 stage ① output
    const std::vector<Cand>& cand1 = C;
    if (out.cand1_ids) {
        for (int32_t j = 0; j < o.ef1; ++j) {
            bool ok = j < (int32_t)cand1.size();
            out.cand1_ids[qi * o.ef1 + j] = ok ? cand1[j].id : -1;
            out.cand1_d[qi * o.ef1 + j] = ok ? cand1[j].d : std::numeric_limits<double>::infinity();
        }
    }
    if (trp) {
        int32_t ne = (int32_t)tr.expand.size(), nv = (int32_t)tr.visit.size();
        out.trace_nexp[qi] = ne;
        out.trace_nvis[qi] = nv;
        for (int32_t j = 0; j < std::min(ne, o.trace_cap); ++j) out.trace_expand[qi * o.trace_cap + j] = tr.expand[j];
        for (int32_t j = 0; j < std::min(nv, o.trace_cap); ++j) out.trace_visit[qi * o.trace_cap + j] = tr.visit[j];
    }

    std::vector<Cand> result;
    if (o.stages == 1) {
        result = cand1;                                        // GPU-only result: top-k of C, δ'
    } else {
        // ---- O8 stage ② residual refinement
        std::vector<Cand> C2;
        VisitedSet vis2;                                        // exact
        for (const Cand& c : cand1) {                           // full δ = primary + residual
            C2.push_back(Cand{dfull(c.id), c.id, false});
            vis2.insert(c.id);
            ++local[kNDist2];
        }
        std::sort(C2.begin(), C2.end(), key_less);
        if (o.flags & 2u) {                                     // O10 no-stage ②
            if ((int32_t)C2.size() > o.ef3) C2.resize(o.ef3);
        } else {
            if ((int32_t)C2.size() > o.ef2) C2.resize(o.ef2);
            greedy(ix.sub_offsets, ix.sub_neighbors, dfull, o.ef2, o.width, o.refine_iters, C2, vis2,
                   local[kNExp2], local[kNDist2], nullptr);
        }
        // ---- O9 stage ③ final traversal on the full graph (Q23)
        std::vector<Cand> C3 = C2;
        for (Cand& c : C3) c.checked = false;                  // carry entries start unchecked
        if ((int32_t)C3.size() > o.ef3) C3.resize(o.ef3);      // capacity ef3 from the start (as O5's resize(ef1))
        greedy(ix.full_offsets, ix.full_neighbors, dfull, o.ef3, o.width, -1, C3, vis2,
               local[kNExp3], local[kNDist3], nullptr);
        result = C3;
    }
    for (int32_t j = 0; j < o.k; ++j) {                        // Q26: pad (−1, +inf)
        bool ok = j < (int32_t)result.size();
        out.out_ids[qi * o.k + j] = ok ? result[j].id : -1;
        out.out_d[qi * o.k + j] = ok ? result[j].d : std::numeric_limits<double>::infinity();
    }
    if (cnt) std::memcpy(cnt, local, sizeof(local));
}

template <class F>
void parallel_for(int64_t m, int32_t threads, F f) {
    int32_t T = threads > 0 ? threads : (int32_t)std::max(1u, std::thread::hardware_concurrency());
    if (T > m) T = (int32_t)std::max<int64_t>(1, m);
    std::vector<std::thread> pool;
    for (int32_t t = 0; t < T; ++t)
        pool.emplace_back([=]() { for (int64_t i = t; i < m; i += T) f(i); });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int orc_version() { return 2; }

// O1 alone: q̂[m][D] = q·V in fp64.
void orc_project(const float* Q, int64_t m, int32_t D, const float* V, double* Qh) {
    for (int64_t r = 0; r < m; ++r)
        for (int32_t j = 0; j < D; ++j) {
            double s = 0.0;
            for (int32_t i = 0; i < D; ++i) s += (double)Q[r * D + i] * (double)V[(int64_t)i * D + j];
            Qh[r * D + j] = s;
        }
}

// O1-O9 for a batch of m queries.
int orc_search(const OrcIndex* ix, const float* Q, int64_t m, const OrcOpts* o, const OrcOut* out) {
    if (!ix || !Q || !o || !out || !out->out_ids || !out->out_d) return -1;
    if (o->stages != 1 && (!ix->rotated || !ix->full_offsets)) return -7;
    parallel_for(m, o->threads, [&](int64_t i) { search_one(*ix, Q + i * ix->dim, *o, *out, i); });
    return 0;
}

// O11: exact top-k by (δ, id) of fp64 queries Qh[m][qstride] (first `dim`
// columns used) over rows `ids` (all n rows if ids == NULL) of X[n][xstride]
// (first `dim` columns used).  Pads with (−1, +inf).
void orc_brute_force(const double* Qh, int64_t m, int32_t qstride, const float* X, int64_t n,
                     int32_t xstride, int32_t dim, const int32_t* ids, int64_t nids, int32_t k,
                     int32_t metric, int32_t threads, int32_t* out_ids, double* out_d) {
    parallel_for(m, threads, [&](int64_t qi) {
        std::vector<Cand> all;
        int64_t cnt = ids ? nids : n;
        all.reserve(cnt);
        for (int64_t j = 0; j < cnt; ++j) {
            int32_t v = ids ? ids[j] : (int32_t)j;
            all.push_back(Cand{delta(Qh + qi * qstride, X + (int64_t)v * xstride, dim, metric), v, false});
        }
        std::sort(all.begin(), all.end(), key_less);
        for (int32_t j = 0; j < k; ++j) {
            bool ok = j < (int32_t)all.size();
            out_ids[qi * k + j] = ok ? all[j].id : -1;
            out_d[qi * k + j] = ok ? all[j].d : std::numeric_limits<double>::infinity();
        }
    });
}

// O14: two-hop entry selection — the baseline of §6.3 "FES analysis" (P:L986-989:
// "the first 2-hop traversal of HNSW as the baseline, both evaluated on the GPU").
// DESIGN.md reading Q30: from the fixed entry node e0 (hop 0) every neighbour of
// e0 is visited (hop 1); then the `beam` hop-1 nodes with the smallest keys
// (δ', id) are expanded in key order and their unvisited neighbours visited
// (hop 2).  Each node is visited once (exact set, e0 included).  Entries = the E
// smallest keys over all visited nodes, e0 included, ascending; padded (−1, +inf).
// Queries are projected as in O1 and δ' is O2 over the reduced rows, on the
// subgraph.
void orc_two_hop(const OrcIndex* ix, const float* Q, int64_t m, int32_t e0, int32_t beam, int32_t E,
                 int32_t threads, int32_t* out_ids, double* out_d, int64_t* n_dist) {
    parallel_for(m, threads, [&](int64_t qi) {
        const int32_t D = ix->dim, dp = ix->rdim;
        std::vector<double> qh(D, 0.0);                        // O1
        for (int32_t j = 0; j < D; ++j) {
            double s = 0.0;
            for (int32_t i = 0; i < D; ++i) s += (double)Q[qi * D + i] * (double)ix->basis[(int64_t)i * D + j];
            qh[j] = s;
        }
        const int64_t rs = ix->reduced_stride ? ix->reduced_stride : dp;
        auto dprime = [&](int32_t v) { return delta(qh.data(), ix->reduced + (int64_t)v * rs, dp, ix->metric); };
        std::unordered_set<int32_t> vis;
        std::vector<Cand> all;                                 // every visited node with its key
        vis.insert(e0);
        all.push_back(Cand{dprime(e0), e0, false});
        std::vector<Cand> hop1;
        for (int64_t e = ix->sub_offsets[e0]; e < ix->sub_offsets[e0 + 1]; ++e) {
            const int32_t v = ix->sub_neighbors[e];
            if (vis.insert(v).second) hop1.push_back(Cand{dprime(v), v, false});
        }
        all.insert(all.end(), hop1.begin(), hop1.end());
        std::sort(hop1.begin(), hop1.end(), key_less);
        for (int32_t j = 0; j < beam && j < (int32_t)hop1.size(); ++j) {
            const int32_t u = hop1[j].id;
            for (int64_t e = ix->sub_offsets[u]; e < ix->sub_offsets[u + 1]; ++e) {
                const int32_t v = ix->sub_neighbors[e];
                if (vis.insert(v).second) all.push_back(Cand{dprime(v), v, false});
            }
        }
        std::sort(all.begin(), all.end(), key_less);
        if (n_dist) n_dist[qi] = (int64_t)all.size();
        for (int32_t j = 0; j < E; ++j) {
            const bool ok = j < (int32_t)all.size();
            out_ids[qi * E + j] = ok ? all[j].id : -1;
            out_d[qi * E + j] = ok ? all[j].d : std::numeric_limits<double>::infinity();
        }
    });
}

// O12: mean over queries of |ret_k ∩ gt_k| / k.  ret[m][rs], gt[m][gs].
// If gt_d and ret_d are given (tie-aware variant, Q25), a returned id counts
// when its δ ≤ δ(gt_k[k−1]) — each returned id at most once.
double orc_recall(const int32_t* ret, int32_t rs, const int32_t* gt, int32_t gs, int64_t m, int32_t k,
                  const double* ret_d, const double* gt_d) {
    double tot = 0.0;
    for (int64_t q = 0; q < m; ++q) {
        int32_t hit = 0;
        for (int32_t a = 0; a < k; ++a) {
            int32_t id = ret[q * rs + a];
            if (id < 0) continue;
            bool dup = false;
            for (int32_t b = 0; b < a; ++b) dup = dup || ret[q * rs + b] == id;
            if (dup) continue;
            if (ret_d && gt_d) {
                if (ret_d[q * rs + a] <= gt_d[q * gs + k - 1]) ++hit;
            } else {
                for (int32_t b = 0; b < k; ++b)
                    if (gt[q * gs + b] == id) { ++hit; break; }
            }
        }
        tot += (double)std::min(hit, k) / (double)k;
    }
    return m > 0 ? tot / (double)m : 0.0;
}

}  // extern "C"
