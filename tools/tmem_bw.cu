// tmem_bw.cu -- dev microbenchmark (sm_100a): throughput of tensor memory used as per-warp accumulator
// storage -- each warp repeatedly loads 4 x 16 columns of its lane quarter (tcgen05.ld 32x32b.x16),
// adds 1 and stores them back (tcgen05.st), as a compositor would per 16-entry chunk if its 64 x 32 fp32
// accumulators lived in TMEM between mma.sync chunks.  CTAs of 4 warps, 64 TMEM columns per CTA,
// k CTAs per SM.  Prints per-SM load+store bytes per cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

template <int MODE>   // 0: ld+st per m-tile (serial wait), 1: 4 lds then 4 sts (one wait each)
__global__ void __launch_bounds__(128) k_tmem(int iters, float* out, unsigned long long* cyc) {
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_taddr)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t r[4][16];
    for (int m = 0; m < 4; m++)
        for (int i = 0; i < 16; i++) r[m][i] = __float_as_uint(0.0f);
    for (int m = 0; m < 4; m++) st16(base + 16 * m, r[m]);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (MODE == 0) {
#pragma unroll
            for (int m = 0; m < 4; m++) {
                uint32_t v[16];
                ld16(base + 16 * m, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; i++) v[i] = __float_as_uint(__uint_as_float(v[i]) + 1.0f);
                st16(base + 16 * m, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else {
            uint32_t v[4][16];
#pragma unroll
            for (int m = 0; m < 4; m++) ld16(base + 16 * m, v[m]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int m = 0; m < 4; m++)
#pragma unroll
                for (int i = 0; i < 16; i++) v[m][i] = __float_as_uint(__uint_as_float(v[m][i]) + 1.0f);
#pragma unroll
            for (int m = 0; m < 4; m++) st16(base + 16 * m, v[m]);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    const unsigned long long t1 = clock64();
    uint32_t v[16];
    ld16(base, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if ((threadIdx.x & 31) == 0) {
        out[blockIdx.x * 4 + warp] = __uint_as_float(v[0]);
        cyc[blockIdx.x * 4 + warp] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(s_taddr) : "memory");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sms * 8 * 4 * sizeof(float));
    cudaMalloc(&cyc, sms * 8 * 4 * sizeof(unsigned long long));
    for (int mode = 0; mode < 2; mode++) {
        for (int k = 1; k <= 8; k *= 2) {
            const int grid = sms * k;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            if (mode == 0) k_tmem<0><<<grid, 128>>>(10, out, cyc); else k_tmem<1><<<grid, 128>>>(10, out, cyc);
            cudaEventRecord(a);
            if (mode == 0) k_tmem<0><<<grid, 128>>>(iters, out, cyc); else k_tmem<1><<<grid, 128>>>(iters, out, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaError_t e = cudaGetLastError();
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long hc[4];
            cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
            const double bytes_per_sm = (double)k * 4 * iters * 4 * 2 * 2048.0;   // warps x iters x mtiles x (ld+st) x 2 KB
            printf("{\"mode\": %d, \"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"ms\": %.4f, \"warp_cycles_per_iter\": %.1f, "
                   "\"ld_st_bytes_per_sm_cycle\": %.1f, \"err\": \"%s\"}\n",
                   mode, k, 4 * k, ms, (double)hc[0] / iters, bytes_per_sm / ((double)hc[0]), cudaGetErrorString(e));
        }
    }
    return 0;
}
