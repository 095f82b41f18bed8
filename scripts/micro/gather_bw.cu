// Random-row gather bandwidth on this GPU: the practical ceiling of the traversal's
// access pattern (independent random rows of B bytes from a multi-GB table), as
// opposed to the sequential copy bandwidth in MEASURED_PEAKS.json.
// usage: gather_bw [table_GB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}

// one row per lane (lane-per-row, like the traversal's distance step), NV float4 per row
template <int NV>
__global__ void k_lane_rows(const float4* __restrict__ t, long long nrows, int iters, float* out) {
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const long long r = (long long)(mix(gt * 1315423911ULL + it) % (unsigned long long)nrows);
        const float4* p = t + r * NV;
        float4 v[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = __ldg(p + i);
#pragma unroll
        for (int i = 0; i < NV; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

// one row per group of NV lanes (coalesced row), NV float4 per row
template <int NV>
__global__ void k_coop_rows(const float4* __restrict__ t, long long nrows, int iters, float* out) {
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long grp = gt / NV;
    const int j = (int)(gt % NV);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const long long r = (long long)(mix(grp * 1315423911ULL + it) % (unsigned long long)nrows);
        const float4 v = __ldg(t + r * NV + j);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) out[0] = acc;
}

// one row per group of L lanes, each lane F = NV/L float4 (lane j reads float4 k*L + j):
// L*16 contiguous bytes per row per load instruction
template <int NV, int L>
__global__ void k_group_rows(const float4* __restrict__ t, long long nrows, int iters, float* out) {
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long grp = gt / L;
    const int j = (int)(gt % L);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const long long r = (long long)(mix(grp * 1315423911ULL + it) % (unsigned long long)nrows);
        float4 v[NV / L];
#pragma unroll
        for (int k = 0; k < NV / L; ++k) v[k] = __ldg(t + r * NV + k * L + j);
#pragma unroll
        for (int k = 0; k < NV / L; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

// rows of STRIDE float4, only the first NV read, by L lanes (lane j: float4 k*L + j < NV)
template <int STRIDE, int NV, int L>
__global__ void k_strided_rows(const float4* __restrict__ t, long long nrows, int iters, float* out) {
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long grp = gt / L;
    const int j = (int)(gt % L);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        const long long r = (long long)(mix(grp * 1315423911ULL + it) % (unsigned long long)nrows);
        float4 v[(NV + L - 1) / L];
#pragma unroll
        for (int k = 0; k < (NV + L - 1) / L; ++k)
            v[k] = (k * L + j < NV) ? __ldg(t + r * STRIDE + k * L + j) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < (NV + L - 1) / L; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

template <class K>
void run(const char* name, K kern, const float4* t, long long nrows, int row_bytes, int grid, int block, int iters,
         long long rows_per_thread_div) {
    float* out;
    cudaMalloc(&out, 4);
    kern<<<grid, block>>>(t, nrows, 2, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<grid, block>>>(t, nrows, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double rows = (double)grid * block / rows_per_thread_div * iters;
    printf("%-28s row %4d B  grid %6d x %4d  %8.1f GB/s  (%.3f ms)\n", name, row_bytes, grid, block,
           rows * row_bytes / (ms * 1e-3) / 1e9, ms);
    cudaFree(out);
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 2.0;
    const size_t bytes = (size_t)(gb * (1ull << 30));
    float4* t;
    if (cudaMalloc(&t, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(t, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("table %.1f GB, %d SMs\n", gb, sms);
    for (int occ : {8, 16}) {
        const int grid = sms * occ;
        run("256B rows L=8 x2 (all)", k_strided_rows<16, 16, 8>, t, bytes / 256, 256, grid, 128, 128, 8);
        run("256B rows L=8 read 192B", k_strided_rows<16, 12, 8>, t, bytes / 256, 192, grid, 128, 128, 8);
        run("256B rows L=16 read 192B", k_strided_rows<16, 12, 16>, t, bytes / 256, 192, grid, 128, 128, 16);
        run("192B rows L=16 (12 act)", k_strided_rows<12, 12, 16>, t, bytes / 192, 192, grid, 128, 128, 16);
        run("128B rows L=8 x1", k_strided_rows<8, 8, 8>, t, bytes / 128, 128, grid, 128, 128, 8);
        run("128B rows L=8 read 96B", k_strided_rows<8, 6, 8>, t, bytes / 128, 96, grid, 128, 128, 8);
        run("96B rows L=8 (6 act)", k_strided_rows<6, 6, 8>, t, bytes / 96, 96, grid, 128, 128, 8);
        run("512B rows L=16 x2", k_strided_rows<32, 32, 16>, t, bytes / 512, 512, grid, 128, 128, 16);
        run("512B rows L=32 x1", k_strided_rows<32, 32, 32>, t, bytes / 512, 512, grid, 128, 128, 32);
        run("lane-per-row 192B (NV=12)", k_lane_rows<12>, t, bytes / 192, 192, grid, 128, 64, 1);
        run("lane-per-row 128B (NV=8)", k_lane_rows<8>, t, bytes / 128, 128, grid, 128, 64, 1);
        run("lane-per-row 96B (NV=6)", k_lane_rows<6>, t, bytes / 96, 96, grid, 128, 64, 1);
        run("lane-per-row 512B (NV=32)", k_lane_rows<32>, t, bytes / 512, 512, grid, 128, 16, 1);
        run("coop 192B (12 lanes)", k_coop_rows<12>, t, bytes / 192, 192, grid, 192, 256, 12);
        run("coop 128B (8 lanes)", k_coop_rows<8>, t, bytes / 128, 128, grid, 128, 256, 8);
        run("group 192B L=4 x3", k_group_rows<12, 4>, t, bytes / 192, 192, grid, 128, 128, 4);
        run("group 192B L=2 x6", k_group_rows<12, 2>, t, bytes / 192, 192, grid, 128, 128, 2);
        run("group 192B L=3 x4", k_group_rows<12, 3>, t, bytes / 192, 192, grid, 96, 128, 3);
        run("group 96B L=2 x3", k_group_rows<6, 2>, t, bytes / 96, 96, grid, 128, 128, 2);
        run("group 256B L=4 x4", k_group_rows<16, 4>, t, bytes / 256, 256, grid, 128, 128, 4);
        run("group 512B L=8 x4", k_group_rows<32, 8>, t, bytes / 512, 512, grid, 128, 128, 8);
        run("group 512B L=4 x8", k_group_rows<32, 4>, t, bytes / 512, 512, grid, 128, 64, 4);
    }
    return 0;
}
