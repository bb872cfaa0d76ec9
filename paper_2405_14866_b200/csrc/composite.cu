// composite.cu -- a6 front-to-back compositing of the C-channel latent feature (sm_100a).
//
// One CTA per 16x16 tile, one pixel per thread; warp w owns pixel rows 2w, 2w+1.
// The tile's (depth, id)-ordered list is consumed in batches of kBatch Gaussians staged in
// shared memory (splat record + feature row converted once to fp32, padded rows so the
// 128-bit staging stores are conflict-free).  While staging, every entry gets an 8-bit mask
// of the warps whose two pixel rows its pixel box touches; each warp then walks only its
// entries (ballot + ffs), so rows a Gaussian cannot reach cost nothing.  Transmittance T,
// the decisions (box, q <= 9, alpha' >= 1/255, T*(1-alpha') < 1e-4) and A = 1 - T follow the
// normative fp32 sequence (DESIGN.md a6) bit for bit; the C accumulators are fp32 FMAs.
// Warps retire when all their pixels stopped (__all_sync); the CTA leaves the list as soon
// as every pixel stopped (__syncthreads_count).
#include "common.cuh"
#include "internal.h"

namespace ta {

constexpr int kBatch = 256;

template <typename FT>
struct FeatLoad;

template <>
struct FeatLoad<float> {
    // row of C floats -> s_row (fp32), 16 B at a time
    template <int C>
    __device__ __forceinline__ static void row(const float* __restrict__ src, float* __restrict__ dst) {
#pragma unroll
        for (int c = 0; c < C; c += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + c));
            *reinterpret_cast<float4*>(dst + c) = v;
        }
    }
};

template <>
struct FeatLoad<__half> {
    template <int C>
    __device__ __forceinline__ static void row(const __half* __restrict__ src, float* __restrict__ dst) {
#pragma unroll
        for (int c = 0; c < C; c += 8) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + c));
            const __half2* h = reinterpret_cast<const __half2*>(&v);
            const float2 a = __half22float2(h[0]), b = __half22float2(h[1]);
            const float2 d = __half22float2(h[2]), e = __half22float2(h[3]);
            *reinterpret_cast<float4*>(dst + c) = make_float4(a.x, a.y, b.x, b.y);
            *reinterpret_cast<float4*>(dst + c + 4) = make_float4(d.x, d.y, e.x, e.y);
        }
    }
};

template <int C, typename FT>
__global__ void __launch_bounds__(256) k_composite(const uint4* __restrict__ rec, const FT* __restrict__ feat,
                                                   const uint32_t* __restrict__ list,
                                                   const uint32_t* __restrict__ offs, uint32_t P, int TX, int W,
                                                   int H, RasterConsts rc, float* __restrict__ Fout,
                                                   float* __restrict__ Aout, int32_t* __restrict__ ncontrib) {
    constexpr int CP = C + 4;   // padded fp32 feature row in smem
    extern __shared__ __align__(16) unsigned char smem[];
    float4* s_g = reinterpret_cast<float4*>(smem);                       // mx, my, ca, cb2
    float2* s_g2 = reinterpret_cast<float2*>(s_g + kBatch);              // cc, alpha
    uint2* s_rect = reinterpret_cast<uint2*>(s_g2 + kBatch);             // x0|x1<<16, y0|y1<<16
    uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_rect + kBatch);     // warp bits
    float* s_f = reinterpret_cast<float*>(s_mask + kBatch);              // [kBatch][CP]

    const int tile = blockIdx.x;
    const int tyi = tile / TX, txi = tile - tyi * TX;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = txi * kTile + lx, py = tyi * kTile + ly;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const float pxf = (float)px, pyf = (float)py;
    const int ty0 = tyi * kTile;

    const uint32_t start = offs[(size_t)tile * P];
    const uint32_t end = offs[(size_t)(tile + 1) * P];

    float F[C];
#pragma unroll
    for (int c = 0; c < C; c++) F[c] = 0.0f;
    float T = 1.0f;
    int nc = 0;
    bool done = (px >= W) || (py >= H);
    bool warp_done = __all_sync(0xffffffffu, done);

    for (uint32_t base = start; base < end; base += kBatch) {
        const int nb = (int)min((uint32_t)kBatch, end - base);
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            const int j = threadIdx.x;
            const uint32_t i = list[base + j];
            const uint4 r0 = rec[2 * i], r1 = rec[2 * i + 1];
            s_g[j] = make_float4(__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z),
                                 __uint_as_float(r0.w));
            s_g2[j] = make_float2(__uint_as_float(r1.x), __uint_as_float(r1.y));
            s_rect[j] = make_uint2(r1.z, r1.w);
            const int y0 = (int)(r1.w & 0xffff), y1 = (int)(r1.w >> 16);
            const int lo = max(y0, ty0) - ty0, hi = min(y1, ty0 + kTile - 1) - ty0;
            uint32_t m = 0;
            if (lo <= hi) m = ((2u << (hi >> 1)) - 1u) & ~((1u << (lo >> 1)) - 1u);
            s_mask[j] = m;
            FeatLoad<FT>::template row<C>(feat + (size_t)i * C, s_f + j * CP);
        }
        __syncthreads();
        if (!warp_done) {
            for (int g = 0; g < nb && !warp_done; g += 32) {
                uint32_t bits = __ballot_sync(0xffffffffu, (g + (int)lane < nb) && ((s_mask[g + lane] >> warp) & 1u));
                while (bits) {
                    const int j = g + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const float4 G = s_g[j];
                    const float2 G2 = s_g2[j];
                    const uint2 rr = s_rect[j];
                    if (!done) {
                        const bool inside = px >= (int)(rr.x & 0xffff) && px <= (int)(rr.x >> 16) &&
                                            py >= (int)(rr.y & 0xffff) && py <= (int)(rr.y >> 16);
                        if (inside) {
                            const float dx = fsub(pxf, G.x), dy = fsub(pyf, G.y);
                            const float q = ffma(ffma(G.z, dx, fmul(G.w, dy)), dx, fmul(fmul(G2.x, dy), dy));
                            if (q <= rc.q_max) {
                                const float e = exp_det(fmul(-0.5f, q));
                                const float a = fminf(rc.alpha_max, fmul(G2.y, e));
                                if (a >= rc.alpha_min) {
                                    const float Tn = fmul(T, fsub(1.0f, a));
                                    if (Tn < rc.t_eps) {
                                        done = true;
                                    } else {
                                        const float w = fmul(a, T);
                                        const float* fr = s_f + j * CP;
#pragma unroll
                                        for (int c = 0; c < C; c += 4) {
                                            const float4 f4 = *reinterpret_cast<const float4*>(fr + c);
                                            F[c + 0] = fmaf(f4.x, w, F[c + 0]);
                                            F[c + 1] = fmaf(f4.y, w, F[c + 1]);
                                            F[c + 2] = fmaf(f4.z, w, F[c + 2]);
                                            F[c + 3] = fmaf(f4.w, w, F[c + 3]);
                                        }
                                        T = Tn;
                                        nc++;
                                    }
                                }
                            }
                        }
                    }
                    if (__all_sync(0xffffffffu, done)) {
                        warp_done = true;
                        break;
                    }
                }
            }
        }
        if (__syncthreads_count(!done) == 0) break;
    }

    if (px < W && py < H) {
        const size_t pix = (size_t)py * W + px;
        float* out = Fout + pix * C;
#pragma unroll
        for (int c = 0; c < C; c += 4) *reinterpret_cast<float4*>(out + c) = make_float4(F[c], F[c + 1], F[c + 2], F[c + 3]);
        Aout[pix] = fsub(1.0f, T);
        if (ncontrib) ncontrib[pix] = nc;
    }
}

template <int C, typename FT>
static cudaError_t launch_one(int tiles, const uint4* rec, const void* feat, const uint32_t* list,
                              const uint32_t* offs, uint32_t P, int TX, int W, int H, RasterConsts rc, float* F,
                              float* A, int32_t* ncontrib, cudaStream_t st) {
    const size_t smem = (size_t)kBatch * (16 + 8 + 8 + 4) + (size_t)kBatch * (C + 4) * sizeof(float);
    static bool attr_set = false;   // per template instance; set once per process
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_composite<C, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (tiles == 0) return cudaSuccess;
    k_composite<C, FT><<<tiles, 256, smem, st>>>(rec, static_cast<const FT*>(feat), list, offs, P, TX, W, H, rc, F,
                                                 A, ncontrib);
    return cudaGetLastError();
}

cudaError_t launch_composite(int C, int fbytes, int tiles, int, const uint4* rec, const void* feat,
                             const uint32_t* list, const uint32_t* offs, uint32_t P, int TX, int W, int H,
                             RasterConsts rc, float* F, float* A, int32_t* ncontrib, cudaStream_t st) {
#define TA_CASE(CC)                                                                                           \
    case CC:                                                                                                  \
        return fbytes == 2 ? launch_one<CC, __half>(tiles, rec, feat, list, offs, P, TX, W, H, rc, F, A, ncontrib, st) \
                           : launch_one<CC, float>(tiles, rec, feat, list, offs, P, TX, W, H, rc, F, A, ncontrib, st);
    switch (C) {
        TA_CASE(8)
        TA_CASE(16)
        TA_CASE(32)
        TA_CASE(64)
        default:
            return cudaErrorInvalidValue;
    }
#undef TA_CASE
}

}  // namespace ta
