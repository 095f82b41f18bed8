// a1 + a2 — query projection and FES routing on the 5th-gen tensor cores.
//
//   [route | q' | q_res] = Q · B_Tᵀ,   B_T = [ (V[:, :d']·Cᵀ)ᵀ ; V[:, :d']ᵀ ; V[:, d':]ᵀ ]   (rows K-major)
//
// q̂ = q·V is P:L244-245 (§4.1 ①); the routing columns are q'·c = q·(V_{:d'}·c)
// so that cell(q) = argmin_c (‖c‖² − 2 q'·c) [L2] or argmin_c (−q'·c) [IP]
// falls out of the same GEMM (SURVEY §8.a a2 "fusion option").
//
// Precision: 3xTF32: a = a_hi + a_lo with a_hi = a truncated to
// TF32, a_lo = a − a_hi (exact); D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi with fp32
// accumulation in TMEM (kind::tf32).  Error ≈ fp32 SIMT (plain TF32 fails 1e-5).
//
// Structure: grid = (128-query tiles) × (column tiles of ≤ 256, multiples of 16;
// the first tile holds the r routing columns, so the argmin stays in one CTA) —
// enough CTAs to cover the 148 SMs at 10K queries.  4 warps per CTA, K loop in
// 32-float chunks through an S-stage smem ring:
//   * B (constant) is pre-split at build into hi/lo planes already in K-major
//     SWIZZLE_128B order (`DevIndex::proj_img`); thread 0 streams each chunk's
//     [n0, n0+w) rows — one contiguous range per plane — with TMA bulk copies
//     (cp.async.bulk → UBLKCP) completing on the stage's `full` mbarrier;
//   * A (the queries) is read with coalesced float4 loads one chunk ahead of its
//     use (registers), split hi/lo and stored swizzled;
//   * thread 0 waits for the stage, issues 4 k-steps × 3 tcgen05.mma (M = 128,
//     N = w, K = 8) and commits to the stage's `empty` mbarrier, which frees the
//     stage S chunks later — loads, splitting and MMAs of different chunks overlap.
// Epilogue: tcgen05.ld 32x32b (thread = query row) → routing argmin (tile 0), q'
// (zero-padded to d'_pad) and q_res.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "internal.h"
#include "umma.cuh"

namespace pa {

namespace {

constexpr int kM = 128;        // UMMA M (queries per CTA)
constexpr int kKC = 32;        // K floats per chunk (128 B, one swizzle atom column)
constexpr int kThreads = 128;
constexpr int kMaxStages = 4;

struct ProjParams {
    const float* q;        // [m][D]
    const float* img;      // [kch][2][NB][32] pre-split, pre-swizzled B_T (proj_img)
    const float* cnorm;    // [r] ‖c‖²
    int64_t m;
    int D, dp, dps, r, NB;
    int ncols;             // columns needed: r + d' (GPU only) or r + D
    int w0, w;             // width of tile 0 and of the other tiles (multiples of 16)
    int stages;
    int metric;
    float* qp;             // [m][dps]
    float* qres;           // [m][D−d'] or null
    int32_t* cell;         // [m]
};

template <bool VEC>
__device__ __forceinline__ void load_a(const ProjParams& p, int64_t row0, int k0, int tid, float4 (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int f = tid + i * kThreads;               // float4 index in the 128 × 8 chunk
        const int row = f >> 3, c4 = f & 7;
        const int64_t gr = row0 + row;
        const int k = k0 + c4 * 4;
        if (VEC) {
            r[i] = (gr < p.m && k < p.D) ? __ldg(reinterpret_cast<const float4*>(p.q + gr * p.D + k))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const float* src = p.q + gr * p.D;
            const bool ok = gr < p.m;
            r[i].x = ok && k + 0 < p.D ? __ldg(src + k + 0) : 0.f;
            r[i].y = ok && k + 1 < p.D ? __ldg(src + k + 1) : 0.f;
            r[i].z = ok && k + 2 < p.D ? __ldg(src + k + 2) : 0.f;
            r[i].w = ok && k + 3 < p.D ? __ldg(src + k + 3) : 0.f;
        }
    }
}

__device__ __forceinline__ void store_a(unsigned char* a_hi, unsigned char* a_lo, int tid, const float4 (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int f = tid + i * kThreads;
        const int row = f >> 3, c4 = f & 7;
        float4 h, l;
        split_tf32(r[i].x, h.x, l.x);
        split_tf32(r[i].y, h.y, l.y);
        split_tf32(r[i].z, h.z, l.z);
        split_tf32(r[i].w, h.w, l.w);
        const uint32_t off = sw128_off(row, c4 * 4);
        *reinterpret_cast<float4*>(a_hi + off) = h;
        *reinterpret_cast<float4*>(a_lo + off) = l;
    }
}

// Dynamic smem: stages × { A_hi | A_lo (16 KB each) | B_hi | B_lo (w_max × 128 B each) }, then
// full[S] | empty[S] mbarriers, tmem slot.
template <bool VEC>
__global__ void __launch_bounds__(kThreads, 1) k_project_tc(ProjParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int tile = blockIdx.y;
    const int n0 = tile == 0 ? 0 : p.w0 + (tile - 1) * p.w;
    const int w = tile == 0 ? p.w0 : min(p.w, ((p.ncols + 15) & ~15) - n0);
    const int wmax = max(p.w0, p.w);
    const uint32_t bplane = (uint32_t)w * 128;
    const uint32_t stage_bytes = 32768u + 2u * (uint32_t)wmax * 128u;
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
    uint64_t* empty = full + S;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + S);

    uint32_t tcols = 32;
    while ((int)tcols < w) tcols <<= 1;
    if (warp == 0) tmem_alloc(tslot, tcols);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tmem = *tslot;

    const int64_t row0 = (int64_t)blockIdx.x * kM;
    const int nch = (p.D + kKC - 1) / kKC;
    const uint32_t idesc = make_idesc_tf32(kM, w);
    float4 ra[8];
    load_a<VEC>(p, row0, 0, tid, ra);
    for (int c = 0; c < nch; ++c) {
        const int s = c % S;
        const uint32_t u = (uint32_t)(c / S);
        unsigned char* st = smem + (size_t)s * stage_bytes;
        unsigned char* a_hi = st;
        unsigned char* a_lo = st + 16384;
        unsigned char* b_hi = st + 32768;
        unsigned char* b_lo = b_hi + (size_t)wmax * 128;
        if (c >= S) mbar_wait(&empty[s], (u - 1) & 1);      // the MMAs of chunk c − S have read this stage
        if (tid == 0) {
            const float* src = p.img + ((size_t)c * 2 * p.NB + n0) * kKC;
            mbar_expect_tx(&full[s], 2 * bplane);
            tma_bulk_g2s(b_hi, src, bplane, &full[s]);
            tma_bulk_g2s(b_lo, src + (size_t)p.NB * kKC, bplane, &full[s]);
        }
        store_a(a_hi, a_lo, tid, ra);
        if (c + 1 < nch) load_a<VEC>(p, row0, (c + 1) * kKC, tid, ra);
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            mbar_wait(&full[s], u & 1);
            tmem_fence_after();
            const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
            const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
#pragma unroll
            for (int kk = 0; kk < kKC / 8; ++kk) {
                const uint32_t koff = (uint32_t)kk * 32;         // 8 tf32 = 32 B along K
                const uint64_t ah = make_desc_sw128(sa_hi + koff), al = make_desc_sw128(sa_lo + koff);
                const uint64_t bh = make_desc_sw128(sb_hi + koff), bl = make_desc_sw128(sb_lo + koff);
                mma_tf32(tmem, ah, bh, idesc, (c > 0 || kk > 0) ? 1u : 0u);
                mma_tf32(tmem, ah, bl, idesc, 1u);
                mma_tf32(tmem, al, bh, idesc, 1u);
            }
            mma_commit(&empty[s]);
        }
    }
    {   // the last commit covers every MMA issued before it
        const int c = nch - 1;
        mbar_wait(&empty[c % S], (uint32_t)(c / S) & 1);
    }
    tmem_fence_after();

    // ---- epilogue: thread = query row = TMEM lane (warp w owns lanes 32w..32w+31)
    const int64_t gr = row0 + tid;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    const int D = p.D;
    float best = __int_as_float(0x7f800000);
    int bestc = 0;
    for (int c0 = 0; c0 < w; c0 += 16) {
        float v[16];
        tmem_ld16(lane_base + (uint32_t)c0, v);
        if (gr < p.m) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int col = n0 + c0 + i;
                if (col < p.r) {
                    const float sc = p.metric == 0 ? fmaf(-2.f, v[i], __ldg(p.cnorm + col)) : -v[i];
                    if (sc < best) { best = sc; bestc = col; }        // strict: tie → lower cell (Q9)
                } else if (col < p.r + p.dp) {
                    p.qp[gr * p.dps + (col - p.r)] = v[i];
                } else if (p.qres && col < p.r + D) {
                    p.qres[gr * (D - p.dp) + (col - p.r - p.dp)] = v[i];
                }
            }
        }
    }
    if (gr < p.m && tile == 0) {
        for (int j = p.dp; j < p.dps; ++j) p.qp[gr * p.dps + j] = 0.f;
        p.cell[gr] = bestc;
    }
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

// Column tiling: tile 0 covers the routing columns; tiles are ≤ 256 wide and the
// grid has ≥ ~148 CTAs when the query tiles alone do not fill the SMs.
void plan_tiles(const DevIndex& ix, int64_t m, bool with_qres, int& ncols, int& w0, int& w, int& ntiles) {
    ncols = ix.fes_r + (with_qres ? ix.dim : ix.rdim);
    const int units = (ncols + 15) / 16;
    const int64_t mt = (m + kM - 1) / kM;
    int nt = (int)std::max<int64_t>(1, (148 + mt - 1) / mt);
    nt = std::max(nt, (units + 15) / 16);                        // ≤ 256 columns per tile
    nt = std::min(nt, units);
    const int ru = (ix.fes_r + 15) / 16;                          // tile 0 holds the routing columns
    int u0 = (units + nt - 1) / nt;
    if (u0 < ru) u0 = std::min(ru, 16);
    int rest = units - u0;
    int nt_rest = nt - 1;
    if (rest <= 0) { nt_rest = 0; rest = 0; }
    int uw = nt_rest > 0 ? (rest + nt_rest - 1) / nt_rest : 1;
    if (uw > 16) { uw = 16; nt_rest = (rest + 15) / 16; }
    w0 = u0 * 16;
    w = uw * 16;
    ntiles = 1 + (rest > 0 ? (rest + uw - 1) / uw : 0);
}

int stages_for(int wmax) {
    const size_t stage = 32768 + (size_t)2 * wmax * 128;
    int S = (int)((200 * 1024) / stage);
    return std::max(2, std::min(kMaxStages, S));
}

}  // namespace

int launch_project_tc(const DevIndex& ix, const SearchArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    ProjParams p;
    p.q = a.q; p.img = ix.proj_img; p.cnorm = ix.cent_norm; p.m = a.m;
    p.D = ix.dim; p.dp = ix.rdim; p.dps = ix.rdim_pad; p.r = ix.fes_r; p.NB = ix.proj_nb; p.metric = ix.metric;
    int ntiles = 1;
    plan_tiles(ix, a.m, a.qres != nullptr, p.ncols, p.w0, p.w, ntiles);
    const int wmax = std::max(p.w0, p.w);
    p.stages = stages_for(wmax);
    p.qp = a.qp; p.qres = a.qres; p.cell = a.cell;
    const size_t smem = (size_t)p.stages * (32768 + (size_t)2 * wmax * 128) + (size_t)16 * p.stages + 16 + 1024;
    dim3 grid((unsigned)((a.m + kM - 1) / kM), (unsigned)ntiles);
    if (ix.dim % 4 == 0) {
        cudaFuncSetAttribute(k_project_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_project_tc<true><<<grid, kThreads, smem, s>>>(p);
    } else {
        cudaFuncSetAttribute(k_project_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_project_tc<false><<<grid, kThreads, smem, s>>>(p);
    }
    return 1;
}

bool project_tc_supported(const DevIndex& ix, bool with_qres) {
    (void)with_qres;
    return ix.proj_img != nullptr && ix.fes_r <= 256;
}

}  // namespace pa
