// a1 — query projection q̂ = q·V, SIMT fp32 first cut.
// The tcgen05 3xTF32 kernel (project_tc.cu) replaces it on the hot path; this
// one stays as the small-m / debugging path and as a cross-check in tests.
#include "internal.h"

namespace pa {

namespace {
constexpr int kQB = 8;   // queries per block

__global__ void __launch_bounds__(256) k_project_simt(const float* __restrict__ q, const float* __restrict__ V,
                                                       int64_t m, int D, int dp, int dps,
                                                       float* __restrict__ qp, float* __restrict__ qres) {
    extern __shared__ float qs[];                    // [kQB][D]
    const int64_t q0 = (int64_t)blockIdx.x * kQB;
    const int nq = (int)((m - q0) < kQB ? (m - q0) : kQB);
    for (int i = threadIdx.x; i < nq * D; i += blockDim.x) qs[i] = q[q0 * D + i];
    __syncthreads();
    const int jmax = qres ? max(D, dps) : dps;
    for (int j = threadIdx.x; j < jmax; j += blockDim.x) {
        float acc[kQB];
#pragma unroll
        for (int t = 0; t < kQB; ++t) acc[t] = 0.f;
        if (j < D) {
            for (int i = 0; i < D; ++i) {
                float v = __ldg(V + (int64_t)i * D + j);
#pragma unroll
                for (int t = 0; t < kQB; ++t) acc[t] = fmaf(qs[t * D + i], v, acc[t]);
            }
        }
        for (int t = 0; t < nq; ++t) {
            if (j < dp) qp[(q0 + t) * dps + j] = acc[t];
            else if (j < dps) qp[(q0 + t) * dps + j] = 0.f;
            if (qres && j >= dp && j < D) qres[(q0 + t) * (D - dp) + (j - dp)] = acc[t];
        }
    }
}
}  // namespace

int launch_project(const DevIndex& ix, const SearchArgs& a, cudaStream_t s) {
    if (a.m == 0) return 0;
    dim3 grid((unsigned)((a.m + kQB - 1) / kQB));
    size_t smem = sizeof(float) * kQB * ix.dim;
    k_project_simt<<<grid, 256, smem, s>>>(a.q, ix.basis, a.m, ix.dim, ix.rdim, ix.rdim_pad, a.qp, a.qres);
    return 1;
}

}  // namespace pa
