// ws_probe2.cu -- TMEM placement of one tcgen05.mma (.ws or not): D[r][n] = 256 r + n (unique); one MMA
// issued by thread 0 at TMEM lane offset LOFF; all 128 lanes x 128 columns read back.  (dev probe)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_fp16.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
__global__ void probe(float* out, int M, int N, int ws, int loff) {
    __shared__ __align__(1024) uint8_t A[2 * 128 * 16];
    __shared__ __align__(1024) uint8_t B[2 * 32 * 128];
    __shared__ uint32_t taddr_s;
    __shared__ __align__(8) unsigned long long bar;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int r = threadIdx.x; r < M; r += 128)
        for (int k = 0; k < 16; k++) {
            float v = k == 0 ? (float)r : k == 1 ? 1.0f : 0.0f;
            *(__half*)&A[(k >> 3) * (M / 8) * 128 + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2] = __float2half(v);
        }
    for (int n = threadIdx.x; n < N; n += 128)
        for (int k = 0; k < 16; k++) {
            float v = k == 0 ? 256.0f : k == 1 ? (float)n : 0.0f;
            *(__half*)&B[(k >> 3) * (N / 8) * 128 + (n >> 3) * 128 + (k & 7) * 16 + (n & 7) * 2] = __float2half(v);
        }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = taddr_s;
    // zero the TMEM region first (tcgen05.st), so untouched cells read as -1
    for (int c0 = 0; c0 < 128; c0++) {
        uint32_t v = __float_as_uint(-1.0f);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + ((uint32_t)(32 * w) << 16) + c0), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (threadIdx.x == 0) {
        const uint64_t ad = sdesc(smem_u32(A), (M / 8) * 128, 128);
        const uint64_t bd = sdesc(smem_u32(B), (N / 8) * 128, 128);
        const uint32_t d = tm + ((uint32_t)loff << 16);
        if (ws)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ad), "l"(bd),
                         "r"(idesc), "r"(0u));
        else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ad), "l"(bd),
                         "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W_%=;\n}\n" ::"r"(
                     smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 128; c0++) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + ((uint32_t)(32 * w) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[(32 * w + l) * 128 + c0] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
int main(int argc, char** argv) {
    const int M = atoi(argv[1]), N = atoi(argv[2]), ws = atoi(argv[3]), loff = atoi(argv[4]);
    float* d;
    cudaMalloc(&d, 128 * 128 * 4);
    probe<<<1, 128>>>(d, M, N, ws, loff);
    cudaError_t e = cudaDeviceSynchronize();
    static float h[128 * 128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=%d N=%d ws=%d lane_off=%d: %s\n", M, N, ws, loff, cudaGetErrorString(e));
    // per lane: the row(s) and column range found
    for (int lane = 0; lane < 128; lane++) {
        int first = -1, last = -1, r0 = -1, nwr = 0;
        for (int c = 0; c < 128; c++) {
            const float v = h[lane * 128 + c];
            if (v >= 0) {
                if (first < 0) { first = c; r0 = (int)v / 256; }
                last = c;
                nwr++;
            }
        }
        if (first >= 0) {
            const float v0 = h[lane * 128 + first], v1 = h[lane * 128 + last];
            printf("  lane %3d: cols %3d..%3d (%3d written)  row %3d n %3d .. row %3d n %3d\n", lane, first, last, nwr,
                   (int)v0 / 256, (int)v0 % 256, (int)v1 / 256, (int)v1 % 256);
        }
    }
    return 0;
}
