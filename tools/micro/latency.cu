// tools/micro/latency.cu -- B200 latency probes for the carry-exchange march
// (diagnostics only; not part of the library).
//   1. dependent DFMA chain (cycles per DFMA)
//   2. dependent double warp shuffle + DFMA (one scan step)
//   3. ping-pong of a 16-byte tagged line between two CTAs on different SMs
//      through L2 (st/ld volatile, as ridc_febe_carry.cuh), round trip cycles
//   4. the same between two warps of one CTA through shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_line(uint4* p, unsigned v, unsigned tag)
{
    asm volatile("st.volatile.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v), "r"(tag), "r"(v), "r"(tag) : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p)
{
    uint4 v;
    asm volatile("ld.volatile.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_line_rel(uint4* p, unsigned v, unsigned tag)
{
    asm volatile("st.relaxed.gpu.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v), "r"(tag), "r"(v), "r"(tag) : "memory");
}
__device__ __forceinline__ uint4 ld_line_rel(const uint4* p)
{
    uint4 v;
    asm volatile("ld.relaxed.gpu.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}

__global__ void k_chain(double* out, long long* cyc, double a, double b)
{
    double x = threadIdx.x, y = 1.0 + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) x = fma(a, x, b);
    long long t1 = clock64();
#pragma unroll 8
    for (int i = 0; i < 256; ++i) {
        const double t = __shfl_up_sync(0xffffffffu, y, 1);
        y = fma(a, t, y);
    }
    long long t2 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0);
        cyc[1] = (t2 - t1);
    }
}

// mode 0: volatile, 1: relaxed.gpu; CTA 0 and CTA 1 ping-pong n times
__global__ void k_pingpong(uint4* lines, long long* cyc, int* smid, int n, int mode)
{
    if (threadIdx.x != 0) return;
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smid[blockIdx.x] = (int)s;
    uint4* mine = lines + blockIdx.x * 8;
    const uint4* other = lines + (1 - blockIdx.x) * 8;
    long long t0 = clock64();
    for (int i = 1; i <= n; ++i) {
        if (blockIdx.x == 0) {
            if (mode == 0) st_line(mine, i, i); else st_line_rel(mine, i, i);
            for (;;) {
                uint4 v = mode == 0 ? ld_line(other) : ld_line_rel(other);
                if (v.y == (unsigned)i && v.w == (unsigned)i) break;
            }
        } else {
            for (;;) {
                uint4 v = mode == 0 ? ld_line(other) : ld_line_rel(other);
                if (v.y == (unsigned)i && v.w == (unsigned)i) break;
            }
            if (mode == 0) st_line(mine, i, i); else st_line_rel(mine, i, i);
        }
    }
    long long t1 = clock64();
    cyc[blockIdx.x] = (t1 - t0) / n;
}

// two warps of one CTA through shared memory
__global__ void k_pingpong_smem(long long* cyc, int n)
{
    __shared__ uint4 s_l[2];
    if (threadIdx.x < 2) s_l[threadIdx.x] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) != 0) return;
    uint4* mine = &s_l[w];
    const uint4* other = &s_l[1 - w];
    long long t0 = clock64();
    for (int i = 1; i <= n; ++i) {
        if (w == 0) {
            st_line(mine, i, i);
            for (;;) {
                uint4 v = ld_line(other);
                if (v.y == (unsigned)i && v.w == (unsigned)i) break;
            }
        } else {
            for (;;) {
                uint4 v = ld_line(other);
                if (v.y == (unsigned)i && v.w == (unsigned)i) break;
            }
            st_line(mine, i, i);
        }
    }
    long long t1 = clock64();
    if (w == 0) cyc[0] = (t1 - t0) / n;
}

int main()
{
    double* out;
    long long* cyc;
    int* smid;
    uint4* lines;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMallocManaged(&cyc, 16 * sizeof(long long));
    cudaMallocManaged(&smid, 16 * sizeof(int));
    cudaMalloc(&lines, 64 * sizeof(uint4));
    k_chain<<<1, 32>>>(out, cyc, 0.999, 1e-3);
    k_chain<<<1, 32>>>(out, cyc, 0.999, 1e-3);
    cudaDeviceSynchronize();
    printf("{\"dfma_chain_cyc\": %.2f, \"shfl_dfma_step_cyc\": %.2f}\n", cyc[0] / 1024.0, cyc[1] / 256.0);
    const int n = 20000;
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(lines, 0, 64 * sizeof(uint4));
        // a large dynamic smem request keeps the two CTAs on different SMs
        cudaFuncSetAttribute(k_pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        k_pingpong<<<2, 32, 200 * 1024>>>(lines, cyc, smid, n, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("{\"pingpong_mode\": \"%s\", \"round_trip_cyc\": %lld, \"smids\": [%d, %d], \"err\": \"%s\"}\n",
               mode == 0 ? "volatile" : "relaxed.gpu", cyc[0], smid[0], smid[1], cudaGetErrorString(e));
    }
    k_pingpong_smem<<<1, 64>>>(cyc, n);
    cudaDeviceSynchronize();
    printf("{\"pingpong_smem_round_trip_cyc\": %lld}\n", cyc[0]);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"clock_khz\": %d}\n", clk);
    return 0;
}
