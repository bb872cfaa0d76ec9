// umma_lat.cu -- latency of (4 x tcgen05.mma M=128 N=32 K=16 + commit -> mbarrier wait), one CTA / many CTAs (dev probe)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
__global__ void lat(long long* out, int iters, int nmma) {
    __shared__ __align__(1024) uint8_t A[4][4096];
    __shared__ __align__(1024) uint8_t B[1024];
    __shared__ uint32_t taddr_s;
    __shared__ __align__(8) unsigned long long bar;
    const int w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) { ((uint32_t*)A)[i] = 0; }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) ((uint32_t*)B)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = taddr_s;
    const uint32_t idesc = (1u << 4) | (1u << 16) | (4u << 17) | (8u << 24);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (threadIdx.x == 0) {
            for (int m = 0; m < nmma; m++) {
                const uint64_t ad = sdesc(smem_u32(&A[m & 3][0]), 2048, 128);
                const uint64_t bd = sdesc(smem_u32(B), 512, 128);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + (m & 1) * 32), "l"(ad),
                             "l"(bd), "r"(idesc), "r"(1u));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        }
        asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}\n" ::"r"(
                         smem_u32(&bar)), "r"((uint32_t)(it & 1)));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}
int main(int argc, char** argv) {
    const int blocks = atoi(argv[1]), nmma = atoi(argv[2]);
    long long* d;
    cudaMalloc(&d, blocks * 8);
    lat<<<blocks, 128>>>(d, 1000, nmma);
    cudaError_t e = cudaDeviceSynchronize();
    long long* h = (long long*)malloc(blocks * 8);
    cudaMemcpy(h, d, blocks * 8, cudaMemcpyDeviceToHost);
    long long s = 0;
    for (int i = 0; i < blocks; i++) s += h[i];
    printf("blocks %d, %d MMAs per commit: %s, mean cycles per (issue+commit+wait) %lld\n", blocks, nmma, cudaGetErrorString(e), s / blocks);
    return 0;
}
