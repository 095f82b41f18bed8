// a5 + a6 launcher: picks the k_traverse variant (traverse_kernel.cuh,
// instantiated in traverse_inst_*.cu) and sizes the persistent grid.
#include "internal.h"

namespace pa {
namespace trav {
void* traverse_pick_0cf(int ef, int d, bool trace);
void* traverse_pick_0wf(int ef, int d, bool trace);
void* traverse_pick_1cf(int ef, int d, bool trace);
void* traverse_pick_1wf(int ef, int d, bool trace);
void* traverse_pick_0ch(int ef, int d, bool trace);
void* traverse_pick_0wh(int ef, int d, bool trace);
void* traverse_pick_1ch(int ef, int d, bool trace);
void* traverse_pick_1wh(int ef, int d, bool trace);
void* traverse_pick_pipe_0cf(int ef, int d, bool trace);
void* traverse_pick_pipe_0ch(int ef, int d, bool trace);
void* traverse_pick_pipe_0wf(int ef, int d, bool trace);
void* traverse_pick_pipe_0wh(int ef, int d, bool trace);
void* traverse_pick_pipe_1cf(int ef, int d, bool trace);
void* traverse_pick_pipe_1ch(int ef, int d, bool trace);
void* traverse_pick_pipe_1wf(int ef, int d, bool trace);
void* traverse_pick_pipe_1wh(int ef, int d, bool trace);
void* traverse_pick_pipe_0bf(int ef, int d, bool trace);
void* traverse_pick_pipe_0bh(int ef, int d, bool trace);
void* traverse_pick_pipe_1bf(int ef, int d, bool trace);
void* traverse_pick_pipe_1bh(int ef, int d, bool trace);

constexpr int kTW = 4;
}  // namespace trav

namespace {
using trav::kTW;

bool use_compact(const DevIndex& ix, const SearchArgs& a) {
    if (a.wide_visited) return false;
    return ix.n <= (1 << 24) && a.hash_log2 >= 11 && a.hash_log2 <= 13;
}
void* pick(const DevIndex& ix, const SearchArgs& a) {
    const bool cp = use_compact(ix, a), tr = a.trace_cap > 0;
    if (a.bloom_log2 > 0) {                                          // bloom visited set: pipelined kernel only
        if (ix.ell_w != 32 || a.width > 1) return nullptr;
        const bool h = ix.reduced_h != nullptr;
        const int d = h ? ix.rdim_h : ix.rdim_pad;
        if (ix.metric == 0) return h ? trav::traverse_pick_pipe_0bh(a.ef, d, tr) : trav::traverse_pick_pipe_0bf(a.ef, d, tr);
        return h ? trav::traverse_pick_pipe_1bh(a.ef, d, tr) : trav::traverse_pick_pipe_1bf(a.ef, d, tr);
    }
    if (ix.ell_w == 32 && a.width == 1) {                            // software-pipelined kernel
        const bool h = ix.reduced_h != nullptr;
        const int d = h ? ix.rdim_h : ix.rdim_pad;
        if (ix.metric == 0) {
            if (cp) return h ? trav::traverse_pick_pipe_0ch(a.ef, d, tr) : trav::traverse_pick_pipe_0cf(a.ef, d, tr);
            return h ? trav::traverse_pick_pipe_0wh(a.ef, d, tr) : trav::traverse_pick_pipe_0wf(a.ef, d, tr);
        }
        if (cp) return h ? trav::traverse_pick_pipe_1ch(a.ef, d, tr) : trav::traverse_pick_pipe_1cf(a.ef, d, tr);
        return h ? trav::traverse_pick_pipe_1wh(a.ef, d, tr) : trav::traverse_pick_pipe_1wf(a.ef, d, tr);
    }
    if (ix.reduced_h) {
        const int d = ix.rdim_h;
        if (ix.metric == 0) return cp ? trav::traverse_pick_0ch(a.ef, d, tr) : trav::traverse_pick_0wh(a.ef, d, tr);
        return cp ? trav::traverse_pick_1ch(a.ef, d, tr) : trav::traverse_pick_1wh(a.ef, d, tr);
    }
    const int d = ix.rdim_pad;
    if (ix.metric == 0) return cp ? trav::traverse_pick_0cf(a.ef, d, tr) : trav::traverse_pick_0wf(a.ef, d, tr);
    return cp ? trav::traverse_pick_1cf(a.ef, d, tr) : trav::traverse_pick_1wf(a.ef, d, tr);
}

size_t smem_bytes(const DevIndex& ix, const SearchArgs& a) {
    const size_t efp = (size_t)((a.ef + 1) & ~1);
    const size_t vis = a.bloom_log2 > 0 ? ((size_t)3 << (a.bloom_log2 - 3))
                                        : ((size_t)(use_compact(ix, a) ? 2 : 4) << a.hash_log2);
    size_t per_warp = efp * 8 + (size_t)ix.qlen * 4 + 128 + vis;   // + 32 ids of compaction scratch
    return per_warp * kTW;
}
}  // namespace

int traverse_max_warps(const DevIndex& ix, const SearchArgs& a) {
    void* fn = pick(ix, a);
    if (!fn) return 0;
    size_t smem = smem_bytes(ix, a);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kTW * 32, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocks < 1) return 0;
    return blocks * sms * kTW;
}

int launch_traverse(const DevIndex& ix, const SearchArgs& a, int grid_warps, cudaStream_t s) {
    if (a.m == 0) return 0;
    void* fn = pick(ix, a);
    size_t smem = smem_bytes(ix, a);
    int64_t want = (a.m + kTW - 1) / kTW;
    int64_t blocks = grid_warps / kTW;
    if (blocks > want) blocks = want;
    if (blocks < 1) blocks = 1;
    cudaMemsetAsync(a.work, 0, sizeof(int32_t), s);
    SearchArgs aa = a;
    DevIndex ii = ix;
    void* args[] = {&ii, &aa};
    cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(kTW * 32), args, smem, s);
    return 1;
}

}  // namespace pa
