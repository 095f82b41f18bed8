// Internal launch interfaces between the runtime (pilotann.cpp) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pa {

// Device-resident replica of one index (SURVEY §8.a layouts).
struct DevIndex {
    int64_t n = 0;
    int32_t dim = 0, rdim = 0, rdim_pad = 0;   // row stride of reduced vectors (multiple of 4 floats)
    int32_t ell_w = 32;                        // ELL row width (32 or 64), −1 padded
    int32_t metric = 0;                        // 0 L2, 1 IP
    int32_t fes_r = 0;
    int64_t pool_n = 0;
    float* basis = nullptr;                    // [dim][dim] row-major V
    float* reduced = nullptr;                  // [n][rstride] (first rdim_pad used; non-members: zero rows); null in fp16 mode
    void* reduced_h = nullptr;                 // [n][rstride_h] binary16 rows (NEXT-f1 storage), first rdim_h = round8(d') used
    int32_t rdim_h = 0;
    int32_t qlen = 0;                          // q' length staged in smem by the traversal (≥ row length)
    int32_t rstride = 0;                       // row stride of `reduced` in floats: multiple of 32 (128-B lines)
    int32_t rstride_h = 0;                     // row stride of `reduced_h` in halves: multiple of 64 (128-B lines)
    int32_t* ell = nullptr;                    // [n][ell_w]
    float* centroids = nullptr;                // [r][rdim_pad]
    int32_t* cell_off = nullptr;               // [r+1]
    int32_t* pool_ids = nullptr;               // [pool_n] grouped by cell
    float* pool_vec = nullptr;                 // [pool_n][rdim_pad] contiguous by cell
    float* proj_img = nullptr;                 // [ceil(dim/32)][hi,lo][proj_nb][32] B_T of the tcgen05 projection,
                                               // split to TF32 hi/lo, rows K-major SWIZZLE_128B (TMA bulk sources)
    int32_t proj_nb = 0;                       // rows of B_T: roundup16(r + dim)
    float* cent_norm = nullptr;                // [r] ‖centroid‖²
    float* pool_norm = nullptr;                // [pool_n] ‖e‖² (GEMM-form FES scores)
    int32_t max_cell = 0;                      // largest FES cell (score scratch row stride, multiple of 4)
    float* pool_img = nullptr;                 // [chunks][kch][hi,lo][4096]: pool split to TF32 hi/lo and laid
                                               // out as K-major SWIZZLE_128B 128×32 tiles (TMA bulk sources)
    int32_t* chunk_off = nullptr;              // [r+1] first 128-entry pool chunk of each cell
    int32_t pool_chunks = 0;                   // total 128-entry pool chunks (= chunk_off[r])
    // NEXT-f3 (PA_STAGES_FULL_GPU), uploaded on first use from pa_attach_host's arrays
    int32_t* full_ell = nullptr;               // [n][full_w] full graph, −1 padded
    int32_t full_w = 0;
    float* xhat = nullptr;                     // [n][xstride] rotated full vectors X̂ (xstride: D rounded to 32)
    int32_t xstride = 0;
    bool fes_fold_norm = false;                // pool_img rows are [−2e, ‖e‖²] (L2, spare K column) else −2e / −e
};

struct SearchArgs {
    int64_t m = 0;
    int32_t k = 10, ef = 64, E = 64;
    uint32_t flags = 0;
    int32_t hash_log2 = 12;
    int32_t bloom_log2 = 0;        // > 0: stage-① visited set = bloom filter, 3 segments × 2^this bits (NEXT-f1)
    bool wide_visited = false;
    int32_t width = 1;             // search width w (1 = Alg 1; > 1: the sequential kernel, exact visited set)     // force the 32-bit exact visited table (pa_search_opts.check_path test hook)
    const float* q = nullptr;      // [m][dim]
    float* qp = nullptr;           // [m][rdim_pad]  projected q'
    float* qres = nullptr;         // [m][dim − rdim] (optional) residual projection for host stages
    int32_t* cell = nullptr;       // [m]
    bool cell_ready = false;       // routing already computed (by the tcgen05 projection epilogue)
    int32_t* perm = nullptr;       // [m]   queries bucketed by cell (a3)
    int32_t* qoff = nullptr;       // [r+1] per-cell query offsets
    int32_t* toff = nullptr;       // [r+1] per-cell 128-query tile offsets
    float* fes_scores = nullptr;   // [m][max_cell] GEMM-form FES scores (tcgen05 path scratch)
    int32_t* entries = nullptr;    // [m][E]
    int32_t* cand_ids = nullptr;   // [m][ef] (optional)
    float* cand_d = nullptr;       // [m][ef] (optional)
    int32_t* out_ids = nullptr;    // [m][k]
    float* out_d = nullptr;        // [m][k]
    int32_t* counters = nullptr;   // [m][4] (optional)
    int32_t* work = nullptr;       // work counter (device int, zeroed by the launcher)
    uint64_t* spill = nullptr;     // [slots_total] epoch-tagged global overflow hash
    int32_t spill_log2 = 16;       // per-warp slab slots = 2^spill_log2
    int64_t spill_warps = 0;       // number of per-warp slabs available
    uint32_t epoch_base = 1;       // level-2 slot tags: epoch = epoch_base + query index (never 0)
    // trace
    int32_t trace_cap = 0;
    int32_t* trace_expand = nullptr;
    int32_t* trace_visit = nullptr;
    int32_t* trace_nexp = nullptr;
    int32_t* trace_nvis = nullptr;
};

// Stages ②③ on the GPU (NEXT-f3, k_refine).
struct Refine23 {
    int64_t m = 0;
    int32_t k = 10, ef1 = 64, ef2 = 32, ef3 = 64, refine_iters = 2, width = 1;
    uint32_t flags = 0;
    int32_t D = 0, dp = 0, qlen = 0, qp_stride = 0;
    const float* qp = nullptr;          // [m][qp_stride] q'
    const float* qres = nullptr;        // [m][D − d'] q_res
    const int32_t* cand = nullptr;      // [m][ef1] stage-① candidate ids (−1 padded)
    const int32_t* sub_ell = nullptr;   // subgraph ELL
    int32_t sub_w = 32;
    const int32_t* full_ell = nullptr;  // full graph ELL
    int32_t full_w = 32;
    const float* xhat = nullptr;        // [n][xstride] X̂
    int32_t xstride = 0;
    int32_t hash_log2 = 12;
    uint64_t* spill = nullptr;
    int32_t spill_log2 = 16;
    int32_t* work = nullptr;
    int32_t* out_ids = nullptr;         // [m][k] full-space top-k
    float* out_d = nullptr;
    int32_t* counters = nullptr;        // [m][4] n_dist2, n_dist3, 0, status
};
int launch_refine(const DevIndex& ix, const Refine23& a, int grid_warps, cudaStream_t s);

// NEXT-f4: two-hop entry selection (oracle O14), the FES baseline of P:L986-989.
struct TwoHopArgs {
    int64_t m = 0;
    int32_t E = 64, beam = 32, e0 = 0;
    const float* qp = nullptr;          // [m][rdim_pad] q'
    int32_t* entries = nullptr;         // [m][E] ids (−1 padded), ascending keys
    float* entry_d = nullptr;           // [m][E] δ' (optional)
    int32_t* n_dist = nullptr;          // [m] nodes visited (optional)
};
int launch_two_hop(const DevIndex& ix, const TwoHopArgs& a, cudaStream_t s);
bool two_hop_supported(const DevIndex& ix, int E);
int refine_max_warps(const DevIndex& ix, const Refine23& a);

// kernels (each returns the number of kernel launches it enqueued)
int launch_project(const DevIndex& ix, const SearchArgs& a, cudaStream_t s);
int launch_project_tc(const DevIndex& ix, const SearchArgs& a, cudaStream_t s);
bool project_tc_supported(const DevIndex& ix, bool with_qres);
int launch_fes(const DevIndex& ix, const SearchArgs& a, cudaStream_t s);
int launch_fes_tc(const DevIndex& ix, const SearchArgs& a, cudaStream_t s);
bool fes_tc_supported(const DevIndex& ix, int E);
size_t fes_tc_scratch_floats(const DevIndex& ix, int64_t m);
int launch_traverse(const DevIndex& ix, const SearchArgs& a, int grid_warps, cudaStream_t s);
int traverse_max_warps(const DevIndex& ix, const SearchArgs& a);   // resident warps for the launch config

}  // namespace pa
