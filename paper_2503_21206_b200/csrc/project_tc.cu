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
// Structure (one CTA per 128-query tile, 4 warps):
//   K loop in 32-float chunks (one 128-B SWIZZLE_128B atom column): every thread
//   loads fp32 rows, splits hi/lo and stores them K-major, 128-B swizzled, into smem;
//   fence.proxy.async; one elected thread issues 4 k-steps × 3 tcgen05.mma (M=128,
//   N ≤ 256 per instruction, K = 8) into the TMEM accumulator, tcgen05.commit →
//   mbarrier; epilogue: tcgen05.ld 32x32b (thread = query row) → routing argmin,
//   q' (zero-padded to d'_pad), q_res.
#include <cstdint>

#include "common.cuh"
#include "internal.h"
#include "umma.cuh"

namespace pa {

namespace {

constexpr int kM = 128;        // UMMA M (queries per CTA)
constexpr int kKC = 32;        // K floats per smem chunk (128 B, one swizzle atom column)
constexpr int kThreads = 128;

struct ProjParams {
    const float* q;        // [m][D]
    const float* bt;       // [Nb][D]  B_T (rows: r routing, then d' q', then D−d' residual), zero-padded rows
    const float* cnorm;    // [r] ‖c‖²
    int64_t m;
    int D, dp, dps, r;
    int ncols;             // columns computed this launch (multiple of 16): r + d' (GPU only) or r + D
    int metric;
    float* qp;             // [m][dps]
    float* qres;           // [m][D−d'] or null
    int32_t* cell;         // [m]
};

// Dynamic smem: A_hi | A_lo (16 KB each) | B_hi | B_lo (ncols_pad × 128 B each) | mbarrier | tmem slot
__global__ void __launch_bounds__(kThreads, 1) k_project_tc(ProjParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ncols = p.ncols;
    const int bbytes = ncols * 128;
    unsigned char* a_hi = smem;
    unsigned char* a_lo = smem + 16384;
    unsigned char* b_hi = smem + 32768;
    unsigned char* b_lo = b_hi + bbytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(b_lo + bbytes);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

    // TMEM columns: power of two ≥ 32 covering ncols (≤ 512)
    uint32_t tcols = 32;
    while ((int)tcols < ncols) tcols <<= 1;
    if (warp == 0) tmem_alloc(tslot, tcols);
    if (tid == 0) mbar_init(bar, 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    const int64_t row0 = (int64_t)blockIdx.x * kM;
    const int D = p.D;
    const int nchunks = (D + kKC - 1) / kKC;
    uint32_t phase = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int k0 = ch * kKC;
        // ---- stage A (this thread's query row) and B rows, split hi/lo, swizzled
        {
            const int64_t gr = row0 + tid;
            const bool ok = gr < p.m;
            const float* src = p.q + gr * D + k0;
#pragma unroll 8
            for (int k = 0; k < kKC; ++k) {
                float a = (ok && k0 + k < D) ? __ldg(src + k) : 0.f;
                float hi, lo;
                split_tf32(a, hi, lo);
                const uint32_t off = sw128_off(tid, k);
                *reinterpret_cast<float*>(a_hi + off) = hi;
                *reinterpret_cast<float*>(a_lo + off) = lo;
            }
        }
        for (int idx = tid; idx < ncols * kKC; idx += kThreads) {
            const int n = idx / kKC, k = idx % kKC;
            float b = (k0 + k < D) ? __ldg(p.bt + (int64_t)n * D + k0 + k) : 0.f;
            float hi, lo;
            split_tf32(b, hi, lo);
            const uint32_t off = sw128_off(n, k);
            *reinterpret_cast<float*>(b_hi + off) = hi;
            *reinterpret_cast<float*>(b_lo + off) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // ---- one thread issues the MMAs of this chunk
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
            const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
            for (int n0 = 0; n0 < ncols; n0 += 256) {
                const int nn = min(256, ncols - n0);
                const uint32_t idesc = make_idesc_tf32(kM, nn);
                const uint32_t td = tmem + (uint32_t)n0;
#pragma unroll
                for (int kk = 0; kk < kKC / 8; ++kk) {
                    const uint32_t koff = (uint32_t)kk * 32;       // 8 tf32 = 32 B along K
                    const uint32_t boff = (uint32_t)n0 * 128;
                    const uint64_t ah = make_desc_sw128(sa_hi + koff), al = make_desc_sw128(sa_lo + koff);
                    const uint64_t bh = make_desc_sw128(sb_hi + boff + koff), bl = make_desc_sw128(sb_lo + boff + koff);
                    const uint32_t acc0 = (ch > 0 || kk > 0) ? 1u : 0u;
                    mma_tf32(td, ah, bh, idesc, acc0);
                    mma_tf32(td, ah, bl, idesc, 1u);
                    mma_tf32(td, al, bh, idesc, 1u);
                }
            }
            mma_commit(bar);
        }
        __syncwarp();
        mbar_wait(bar, phase);           // MMAs done: smem reusable, accumulator final after last chunk
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    // ---- epilogue: thread = query row = TMEM lane (warp w owns lanes 32w..32w+31)
    const int64_t gr = row0 + tid;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    float best = __int_as_float(0x7f800000);
    int bestc = 0;
    for (int c0 = 0; c0 < ncols; c0 += 16) {
        float v[16];
        tmem_ld16(lane_base + (uint32_t)c0, v);
        if (gr < p.m) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int col = c0 + i;
                if (col < p.r) {
                    const float s = p.metric == 0 ? fmaf(-2.f, v[i], __ldg(p.cnorm + col)) : -v[i];
                    if (s < best) { best = s; bestc = col; }          // strict: tie → lower cell (Q9)
                } else if (col < p.r + p.dp) {
                    p.qp[gr * p.dps + (col - p.r)] = v[i];
                } else if (p.qres && col < p.r + D) {
                    p.qres[gr * (D - p.dp) + (col - p.r - p.dp)] = v[i];
                }
            }
        }
    }
    if (gr < p.m) {
        for (int j = p.dp; j < p.dps; ++j) p.qp[gr * p.dps + j] = 0.f;
        p.cell[gr] = bestc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem_dealloc(tmem, tcols);
    }
}

}  // namespace

int launch_project_tc(const DevIndex& ix, const SearchArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    ProjParams p;
    p.q = a.q; p.bt = ix.proj_bt; p.cnorm = ix.cent_norm; p.m = a.m;
    p.D = ix.dim; p.dp = ix.rdim; p.dps = ix.rdim_pad; p.r = ix.fes_r; p.metric = ix.metric;
    const int need = ix.fes_r + (a.qres ? ix.dim : ix.rdim);
    p.ncols = (need + 15) & ~15;
    p.qp = a.qp; p.qres = a.qres; p.cell = a.cell;
    const size_t smem = 32768 + (size_t)2 * p.ncols * 128 + 16;
    cudaFuncSetAttribute(k_project_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)((a.m + kM - 1) / kM);
    k_project_tc<<<grid, kThreads, smem, s>>>(p);
    return 1;
}

bool project_tc_supported(const DevIndex& ix, bool with_qres) {
    const int need = ix.fes_r + (with_qres ? ix.dim : ix.rdim);
    const int ncols = (need + 15) & ~15;
    return ix.proj_bt != nullptr && ncols <= 512 && 32768 + (size_t)2 * ncols * 128 + 16 <= 227 * 1024;
}

}  // namespace pa
