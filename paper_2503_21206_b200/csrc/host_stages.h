// Host stages ②③ interface (internal).
#pragma once
#include <cstdint>

namespace pa {

struct HostGraph {
    const int64_t* off = nullptr;
    const int32_t* nb = nullptr;
};

struct HostStageArgs {
    int32_t dim = 0, rdim = 0, metric = 0;
    HostGraph sub, full;
    const float* rotated = nullptr;     // X̂ [n][dim]
    int64_t m = 0;
    int32_t k = 10, ef1 = 64, ef2 = 32, ef3 = 64;
    long refine_iters = 2;
    int32_t width = 1;                  // search width w: expansions per Alg 1 iteration
    uint32_t flags = 0;
    int threads = 0;
    const int32_t* cand_ids = nullptr;  // [m][ef1] stage-① C
    const float* cand_d = nullptr;      // [m][ef1] δ' (fp32, from the GPU)
    const float* qp = nullptr;          // [m][qp_stride] q'
    int32_t qp_stride = 0;
    const float* qres = nullptr;        // [m][dim − rdim]
    int32_t* out_ids = nullptr;         // [m][k]
    float* out_d = nullptr;             // [m][k]
    bool recompute_primary = false;     // full δ from X̂ over all D dims instead of δ' + residual
    int64_t* sum_n_dist2 = nullptr;
    int64_t* sum_n_dist3 = nullptr;
    // Optional pipelining hook: called before a worker first touches a query of a
    // new sub-batch (queries are claimed in increasing order), e.g. to wait for the
    // D2H of that sub-batch's candidates.
    void (*wait_ready)(void* ctx, int64_t q) = nullptr;
    void* ready_ctx = nullptr;
};

void run_host_stages(const HostStageArgs& a);

}  // namespace pa
