// NEXT-f4 — two-hop entry selection, the baseline FES is measured against in
// §6.3 "FES analysis" ("the first 2-hop traversal of HNSW as the
// baseline, both evaluated on the GPU").  Oracle O14, reading Q30:
// from the fixed entry node e0, hop 1 visits N(e0); hop 2 visits the neighbours
// of the `beam` hop-1 nodes with the smallest keys (δ', id); every node once;
// entries = the E smallest keys over all visited nodes (e0 included), ascending.
//
// One warp per query (grid-stride over queries).  Per warp in smem: the sorted
// top-E key list (rank-merged as in the traversal), q', 32 ids of compaction
// scratch and an exact open-addressing visited table of 2^12 int32 slots
// (≤ 1 + 32 + 32·32 = 1057 visits for ELL width 32, so it is never more than
// 26 % full).  Distances use the traversal's 4-lanes-per-row group gathers.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pa {
namespace {

constexpr int kHW = 4;              // warps per block
constexpr int kHLog2 = 12;          // visited slots per warp
constexpr int kHL = 4;              // lanes per row in the distance gathers

__device__ __forceinline__ bool th_insert(int32_t* H, int32_t v) {
    constexpr uint32_t mask = (1u << kHLog2) - 1u;
    uint32_t h = ((uint32_t)v * 0x9E3779B1u) >> (32 - kHLog2);
    for (;;) {
        const int32_t cur = reinterpret_cast<volatile int32_t*>(H)[h];
        if (cur == v) return false;
        if (cur == -1) {
            const int32_t old = atomicCAS(&H[h], -1, v);
            if (old == -1) return true;
            if (old == v) return false;
        }
        h = (h + 1) & mask;
    }
}

template <int METRIC, int NVR, int SMAX>
__global__ void __launch_bounds__(kHW * 32) k_two_hop(DevIndex ix, TwoHopArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int E = a.E, Ep = (E + 1) & ~1, dps = ix.rdim_pad, qlen = ix.qlen;
    const size_t per_warp = (size_t)Ep * 8 + (size_t)qlen * 4 + 128 + ((size_t)4 << kHLog2);
    unsigned char* base = smem_raw + per_warp * w;
    uint64_t* C = reinterpret_cast<uint64_t*>(base);
    float* qs = reinterpret_cast<float*>(C + Ep);
    int32_t* scr = reinterpret_cast<int32_t*>(qs + qlen);
    int32_t* H = scr + 32;
    const unsigned lt_mask = (1u << lane) - 1u;
    const unsigned char* rows = reinterpret_cast<const unsigned char*>(ix.reduced);
    const int64_t stride = (int64_t)ix.rstride * 4;
    const int nvr = dps >> 2;
    const int64_t nw = (int64_t)gridDim.x * kHW;

    for (int64_t q = (int64_t)blockIdx.x * kHW + w; q < a.m; q += nw) {
        for (int i = lane; i < qlen; i += 32) qs[i] = i < dps ? a.qp[q * dps + i] : 0.f;
        int4* H4 = reinterpret_cast<int4*>(H);
        for (int i = lane; i < (1 << (kHLog2 - 2)); i += 32) H4[i] = make_int4(-1, -1, -1, -1);
        __syncwarp();
        int csz = 0, n_dist = 0;
        // visit this lane's id (−1 = none); keys of the new ids, compacted to lanes 0..nnew−1
        auto batch = [&](int32_t v) -> uint64_t {
            const bool isnew = v >= 0 && th_insert(H, v);
            const unsigned bal = __ballot_sync(kFull, isnew);
            const int nnew = __popc(bal);
            if (nnew == 0) return kKeyInf;
            n_dist += nnew;
            if (isnew) scr[__popc(bal & lt_mask)] = v;
            __syncwarp();
            const int32_t cid = lane < nnew ? scr[lane] : 0;
            __syncwarp();
            const float d = group_dists<METRIC, NVR, false, kHL, false>(qs, rows, stride, nvr, cid, nnew, lane);
            return lane < nnew ? make_key(d, cid) : kKeyInf;
        };
        auto merge = [&](uint64_t key) {
            const uint64_t thresh = csz == E ? C[E - 1] : kKeyInf;
            const bool pass = key < thresh;
            const unsigned pb = __ballot_sync(kFull, pass);
            if (pb == 0) return;
            int minr;
            csz = rank_merge<SMAX>(C, csz, E, key, pass, pb, lane, minr);
        };
        merge(batch(lane == 0 ? a.e0 : -1));                                      // hop 0
        const uint64_t k1 = batch(__ldg(ix.ell + (int64_t)a.e0 * 32 + lane));     // hop 1
        merge(k1);
        const uint64_t s1 = warp_sort32(k1, lane);                                // hop-1 keys ascending
        for (int j = 0; j < a.beam && j < 32; ++j) {                              // hop 2, in key order
            const uint32_t hi = __shfl_sync(kFull, (uint32_t)(s1 >> 32), j);
            const uint32_t lo = __shfl_sync(kFull, (uint32_t)s1, j);
            const uint64_t kj = ((uint64_t)hi << 32) | lo;
            if (kj == kKeyInf) break;
            merge(batch(__ldg(ix.ell + (int64_t)key_id(kj) * 32 + lane)));
        }
        const float inf = __int_as_float(0x7f800000);
        for (int i = lane; i < E; i += 32) {
            a.entries[q * E + i] = i < csz ? key_id(C[i]) : -1;
            if (a.entry_d) a.entry_d[q * E + i] = i < csz ? key_dist(C[i]) : inf;
        }
        if (lane == 0 && a.n_dist) a.n_dist[q] = n_dist;
        __syncwarp();
    }
}

template <int METRIC, int SMAX>
void* pick_nvr(int nvr) {
    switch (nvr) {
        case 8: return (void*)k_two_hop<METRIC, 8, SMAX>;
        case 12: return (void*)k_two_hop<METRIC, 12, SMAX>;
        case 16: return (void*)k_two_hop<METRIC, 16, SMAX>;
        case 24: return (void*)k_two_hop<METRIC, 24, SMAX>;
        case 32: return (void*)k_two_hop<METRIC, 32, SMAX>;
        default: return (void*)k_two_hop<METRIC, 0, SMAX>;
    }
}
template <int METRIC>
void* pick_e(int E, int nvr) {
    if (E <= 64) return pick_nvr<METRIC, 2>(nvr);
    if (E <= 128) return pick_nvr<METRIC, 4>(nvr);
    return pick_nvr<METRIC, 8>(nvr);
}

}  // namespace

bool two_hop_supported(const DevIndex& ix, int E) {
    return ix.ell_w == 32 && ix.reduced != nullptr && E >= 1 && E <= 256;
}

int launch_two_hop(const DevIndex& ix, const TwoHopArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    void* fn = ix.metric == 0 ? pick_e<0>(a.E, ix.rdim_pad / 4) : pick_e<1>(a.E, ix.rdim_pad / 4);
    const size_t per_warp = (size_t)((a.E + 1) & ~1) * 8 + (size_t)ix.qlen * 4 + 128 + ((size_t)4 << kHLog2);
    const size_t smem = per_warp * kHW;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kHW * 32, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (int64_t)std::max(blocks, 1) * sms;
    const int64_t want = (a.m + kHW - 1) / kHW;
    if (grid > want) grid = want;
    TwoHopArgs aa = a;
    DevIndex ii = ix;
    void* args[] = {&ii, &aa};
    cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kHW * 32), args, smem, s);
    return 1;
}

}  // namespace pa
