// NEXT-f3 launcher: stages ②③ on the GPU (k_refine, traverse_kernel.cuh).
#include "traverse_kernel.cuh"

namespace pa {
namespace trav {
void* refine_pick_m0(int cap, int D, bool compact);   // stages23_inst_m*.cu
void* refine_pick_m1(int cap, int D, bool compact);
}  // namespace trav
namespace {
using trav::kTW;

bool refine_compact(const DevIndex& ix, const Refine23& a) {
    return ix.n <= (1 << 24) && a.hash_log2 >= 11 && a.hash_log2 <= 13;
}

void* pick(const DevIndex& ix, const Refine23& a) {
    const int cap = a.ef2 > a.ef3 ? a.ef2 : a.ef3;
    const bool cp = refine_compact(ix, a);
    return ix.metric == 0 ? trav::refine_pick_m0(cap, a.D, cp) : trav::refine_pick_m1(cap, a.D, cp);
}

size_t smem_bytes(const DevIndex& ix, const Refine23& a) {
    const int cap = a.ef2 > a.ef3 ? a.ef2 : a.ef3;
    const size_t efp = (size_t)((cap + 1) & ~1);
    const size_t per_warp = efp * 8 + (size_t)a.qlen * 4 + 128 +
                            ((size_t)(refine_compact(ix, a) ? 2 : 4) << a.hash_log2);
    return per_warp * kTW;
}
}  // namespace

int refine_max_warps(const DevIndex& ix, const Refine23& a) {
    void* fn = pick(ix, a);
    const size_t smem = smem_bytes(ix, a);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kTW * 32, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return blocks < 1 ? 0 : blocks * sms * kTW;
}

int launch_refine(const DevIndex& ix, const Refine23& a, int grid_warps, cudaStream_t s) {
    if (a.m == 0) return 0;
    void* fn = pick(ix, a);
    const size_t smem = smem_bytes(ix, a);
    int64_t blocks = grid_warps / kTW;
    const int64_t want = (a.m + kTW - 1) / kTW;
    if (blocks > want) blocks = want;
    if (blocks < 1) blocks = 1;
    cudaMemsetAsync(a.work, 0, sizeof(int32_t), s);
    Refine23 aa = a;
    void* args[] = {&aa};
    cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(kTW * 32), args, smem, s);
    return 1;
}

}  // namespace pa
