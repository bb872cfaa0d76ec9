// backward.cu -- SURVEY 8(f) NEXT #4: backward pass of the compositing step (sm_100a).
//
// Gradients of L = sum_p G_F(p) . F(p) + G_A(p) A(p) with respect to each Gaussian's 2D splat
// parameters (mean2, conic (ca, cb2, cc), alpha) and feature row, for the a6 forward of PAPER.md
// l.386-387 (the differentiable rasterizer of [kerbl20233d]); reading R25 (decisions held
// fixed, no gradient through a binding alpha clamp).  It reuses the splat records and the per-tile
// lists of the preceding ta_rasterize on the same context.
// One CTA per 16 x 16 tile, one pixel per thread; the tile list is staged 256 entries at a time in
// shared memory (record + fp32 feature row).  Pass 1 replays the forward per pixel (the same fp32
// decision sequence as the forward kernels, so the composited set is identical) and accumulates
// S = sum w_j g_j (g_j = G_F . f_j) and T_end; pass 2 replays it again and forms every composited
// entry's per-pixel terms: dL/dalpha'_j = T_j g_j - (S - sum_{k<=j} w_k g_k)/(1 - alpha'_j)
// + G_A T_end/(1 - alpha'_j), chained to alpha, q, conic and mean2, and w_j G_F for the features.
// Per entry the 32 pixels of a warp are summed with shuffles and one lane adds them to the global
// gradient arrays (fp32 atomics: the summation order over warps is not fixed).
#include "common.cuh"
#include "internal.h"

namespace ta {

constexpr int kBwdThreads = 256;
constexpr int kBwdBatch = 256;

template <typename FT>
__device__ __forceinline__ float feat_f32(const FT* p);
template <>
__device__ __forceinline__ float feat_f32<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float feat_f32<__half>(const __half* p) { return __half2float(__ldg(p)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int C, typename FT>
__global__ void __launch_bounds__(kBwdThreads) k_composite_bwd(const uint4* __restrict__ rec, const FT* __restrict__ feat,
                                                               const uint32_t* __restrict__ tlist,
                                                               const uint2* __restrict__ trng, CompositeGeom cg,
                                                               RasterConsts rc, const CallState* __restrict__ cs,
                                                               uint64_t list_cap, const float* __restrict__ GF,
                                                               const float* __restrict__ GA, float* __restrict__ d_mean2,
                                                               float* __restrict__ d_conic, float* __restrict__ d_alpha,
                                                               float* __restrict__ d_feat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4* s_g = reinterpret_cast<float4*>(smem_raw);                 // mx, my, ca, cb2
    float4* s_h = s_g + kBwdBatch;                                      // cc, alpha, box x, box y
    uint32_t* s_i = reinterpret_cast<uint32_t*>(s_h + kBwdBatch);      // array index
    float* s_f = reinterpret_cast<float*>(s_i + kBwdBatch);            // [kBwdBatch][C]
    const int tile = blockIdx.x;
    const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
    const uint2 tr = trng[tile];
    const uint32_t start = tr.x;
    uint32_t end = tr.x + tr.y;
    if (end > list_cap) end = (uint32_t)list_cap;
    const uint32_t n = cs->n;
    const int px = txi * kTile + (int)(threadIdx.x & 15), py = tyi * kTile + (int)(threadIdx.x >> 4);
    const bool inside = px < cg.W && py < cg.H;
    const size_t pix = inside ? (size_t)py * cg.W + px : 0;
    const float pxf = (float)px, pyf = (float)py;
    const float qmax = rc.q_max;
    float gf[C];
#pragma unroll
    for (int c = 0; c < C; c++) gf[c] = inside ? GF[pix * C + c] : 0.0f;
    const float ga = inside ? GA[pix] : 0.0f;

    // stage entries [b0, b0 + cnt) of the tile list into shared memory
    auto stage = [&](uint32_t b0, uint32_t cnt) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) {
            const uint32_t i = tlist[b0 + k];
            const uint32_t ii = i < n ? i : 0u;
            const uint4 r0 = rec[2 * ii], r1 = rec[2 * ii + 1];
            s_g[k] = make_float4(__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z), __uint_as_float(r0.w));
            s_h[k] = make_float4(__uint_as_float(r1.x), __uint_as_float(r1.y), __uint_as_float(r1.z), __uint_as_float(r1.w));
            s_i[k] = i;
        }
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < cnt * C; k += blockDim.x) {
            const uint32_t e = k / C, c = k - e * C;
            const uint32_t i = s_i[e] < n ? s_i[e] : 0u;
            s_f[e * C + c] = feat_f32<FT>(feat + (size_t)i * C + c);
        }
        __syncthreads();
    };
    // the a6 decision sequence for entry k of the staged batch: returns alpha' (0 if not taken)
    auto eval = [&](uint32_t k, float* e_out, float* ae_out, float* dx_out, float* dy_out) -> float {
        const float4 G = s_g[k], Hh = s_h[k];
        const uint32_t bx = __float_as_uint(Hh.z), by = __float_as_uint(Hh.w);
        const int x0 = (int)(bx & 0xffff), x1 = (int)(bx >> 16), y0 = (int)(by & 0xffff), y1 = (int)(by >> 16);
        if (s_i[k] >= n || px < x0 || px > x1 || py < y0 || py > y1) return 0.0f;
        const float dx = fsub(pxf, G.x), dy = fsub(pyf, G.y);
        const float q = ffma(ffma(G.z, dx, fmul(G.w, dy)), dx, fmul(fmul(Hh.x, dy), dy));
        if (!(q <= qmax)) return 0.0f;
        const float e = exp_det(fmul(-0.5f, q));
        const float ae = fmul(Hh.y, e);
        const float a = fminf(rc.alpha_max, ae);
        if (a < rc.alpha_min) return 0.0f;
        *e_out = e; *ae_out = ae; *dx_out = dx; *dy_out = dy;
        return a;
    };

    // warp strip: threads 32w .. 32w+31 = pixel rows 2w, 2w+1 of the tile, all 16 columns
    const int sy0 = tyi * kTile + 2 * (int)(threadIdx.x >> 5), sx0 = txi * kTile;
    auto strip_hit = [&](uint32_t k) -> bool {
        const float4 Hh = s_h[k];
        const uint32_t bx = __float_as_uint(Hh.z), by = __float_as_uint(Hh.w);
        return (int)(bx & 0xffff) <= sx0 + 15 && (int)(bx >> 16) >= sx0 && (int)(by & 0xffff) <= sy0 + 1 &&
               (int)(by >> 16) >= sy0;
    };
    // ---- pass 1: forward replay -> S, T_end, the list position after the last composited entry
    float T = 1.0f, S = 0.0f;
    uint32_t stop = start;
    bool done = !inside;
    for (uint32_t b0 = start; b0 < end; b0 += kBwdBatch) {
        if (__syncthreads_and(done)) break;
        const uint32_t cnt = min((uint32_t)kBwdBatch, end - b0);
        stage(b0, cnt);
        for (uint32_t k = 0; k < cnt && !done; k++) {
            if (!strip_hit(k)) continue;                      // warp-uniform: no pixel of the strip in the box
            float e, ae, dx, dy;
            const float a = eval(k, &e, &ae, &dx, &dy);
            if (a == 0.0f) continue;
            const float Tn = fmul(T, fsub(1.0f, a));
            if (Tn < rc.t_eps) { done = true; break; }
            const float w = fmul(a, T);
            float g = 0.0f;
#pragma unroll
            for (int c = 0; c < C; c++) g = ffma(gf[c], s_f[k * C + c], g);
            S = ffma(w, g, S);
            T = Tn;
            stop = b0 + k + 1;
        }
    }
    const float Tend = T;
    // ---- pass 2: gradients
    T = 1.0f;
    float Sup = 0.0f;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wstop = __reduce_max_sync(0xffffffffu, stop);
    const uint32_t bstop_w = wstop;
    __shared__ uint32_t s_stop;
    if (threadIdx.x == 0) s_stop = start;
    __syncthreads();
    atomicMax(&s_stop, bstop_w);
    __syncthreads();
    const uint32_t cta_stop = s_stop;
    for (uint32_t b0 = start; b0 < cta_stop; b0 += kBwdBatch) {
        const uint32_t cnt = min((uint32_t)kBwdBatch, cta_stop - b0);
        stage(b0, cnt);
        for (uint32_t k = 0; k < cnt; k++) {
            if (b0 + k >= wstop) break;                       // warp-uniform
            if (!strip_hit(k)) continue;
            float e = 0.0f, ae = 0.0f, dx = 0.0f, dy = 0.0f;
            float a = (b0 + k < stop) ? eval(k, &e, &ae, &dx, &dy) : 0.0f;
            const bool take = a != 0.0f;
            if (!__any_sync(0xffffffffu, take)) continue;
            float w = 0.0f, dq = 0.0f, dal = 0.0f, g = 0.0f;
            const float4 G = s_g[k], Hh = s_h[k];
            if (take) {
                w = fmul(a, T);
#pragma unroll
                for (int c = 0; c < C; c++) g = ffma(gf[c], s_f[k * C + c], g);
                Sup = ffma(w, g, Sup);
                const float oma = fsub(1.0f, a);
                const float dad = fsub(fmul(T, g), fdiv(fsub(S, Sup), oma)) + fdiv(fmul(ga, Tend), oma);
                if (!(ae > rc.alpha_max)) {
                    dal = fmul(dad, e);
                    dq = fmul(fmul(dad, Hh.y), fmul(-0.5f, e));
                }
                T = fmul(T, oma);
            }
            // per-entry sums over the warp's pixels
            const float s_al = warp_sum(dal);
            const float s_c0 = warp_sum(fmul(fmul(dq, dx), dx));
            const float s_c1 = warp_sum(fmul(fmul(dq, dx), dy));
            const float s_c2 = warp_sum(fmul(fmul(dq, dy), dy));
            const float s_m0 = warp_sum(fmul(dq, -fadd(fmul(fmul(2.0f, G.z), dx), fmul(G.w, dy))));
            const float s_m1 = warp_sum(fmul(dq, -fadd(fmul(G.w, dx), fmul(fmul(2.0f, Hh.x), dy))));
            const uint32_t gi = s_i[k];
            if (lane == 0) {
                atomicAdd(d_alpha + gi, s_al);
                atomicAdd(d_conic + 3 * (size_t)gi + 0, s_c0);
                atomicAdd(d_conic + 3 * (size_t)gi + 1, s_c1);
                atomicAdd(d_conic + 3 * (size_t)gi + 2, s_c2);
                atomicAdd(d_mean2 + 2 * (size_t)gi + 0, s_m0);
                atomicAdd(d_mean2 + 2 * (size_t)gi + 1, s_m1);
            }
            if constexpr (C >= 32) {
                // butterfly reduce-scatter per 32-channel block: after 5 halvings lane l holds the
                // warp sum of channel (block * 32 + l)
#pragma unroll
                for (int cb = 0; cb < C; cb += 32) {
                    float v[32];
#pragma unroll
                    for (int c = 0; c < 32; c++) v[c] = fmul(w, gf[cb + c]);
#pragma unroll
                    for (int h = 16; h >= 1; h >>= 1) {
                        const bool upper = (lane & h) != 0;
#pragma unroll
                        for (int c = 0; c < h; c++) {
                            const float send = upper ? v[c] : v[c + h];
                            const float keep = upper ? v[c + h] : v[c];
                            v[c] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                        }
                    }
                    atomicAdd(d_feat + (size_t)gi * C + cb + lane, v[0]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    const float v = warp_sum(fmul(w, gf[c]));
                    if (lane == (uint32_t)c) atomicAdd(d_feat + (size_t)gi * C + c, v);
                }
            }
        }
    }
}

// Zero the gradient outputs of the first n = cs->n Gaussians (n may be known only on the device).
__global__ void k_bwd_zero(const CallState* __restrict__ cs, int C, float* __restrict__ d_mean2,
                           float* __restrict__ d_conic, float* __restrict__ d_alpha, float* __restrict__ d_feat) {
    const uint32_t n = cs->n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        d_mean2[2 * (size_t)i] = 0.0f; d_mean2[2 * (size_t)i + 1] = 0.0f;
        d_conic[3 * (size_t)i] = 0.0f; d_conic[3 * (size_t)i + 1] = 0.0f; d_conic[3 * (size_t)i + 2] = 0.0f;
        d_alpha[i] = 0.0f;
        for (int c = 0; c < C; c++) d_feat[(size_t)i * C + c] = 0.0f;
    }
}

cudaError_t launch_composite_bwd(int C, int fbytes, int tiles, const uint4* rec, const void* feat, const uint32_t* tlist,
                                 const uint2* trng, CompositeGeom cg, RasterConsts rc, const CallState* cs,
                                 uint64_t list_cap, const float* GF, const float* GA, float* d_mean2, float* d_conic,
                                 float* d_alpha, float* d_feat, cudaStream_t st) {
    const size_t smem = (size_t)kBwdBatch * (16 + 16 + 4 + 4 * (size_t)C);
    k_bwd_zero<<<1184, 256, 0, st>>>(cs, C, d_mean2, d_conic, d_alpha, d_feat);
#define TA_BWD(CC)                                                                                                      \
    case CC: {                                                                                                          \
        if (fbytes == 2) {                                                                                              \
            cudaFuncSetAttribute(k_composite_bwd<CC, __half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
            k_composite_bwd<CC, __half><<<tiles, kBwdThreads, smem, st>>>(rec, static_cast<const __half*>(feat), tlist, \
                                                                          trng, cg, rc, cs, list_cap, GF, GA, d_mean2,  \
                                                                          d_conic, d_alpha, d_feat);                    \
        } else {                                                                                                        \
            cudaFuncSetAttribute(k_composite_bwd<CC, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
            k_composite_bwd<CC, float><<<tiles, kBwdThreads, smem, st>>>(rec, static_cast<const float*>(feat), tlist,   \
                                                                         trng, cg, rc, cs, list_cap, GF, GA, d_mean2,   \
                                                                         d_conic, d_alpha, d_feat);                     \
        }                                                                                                               \
        return cudaGetLastError();                                                                                      \
    }
    switch (C) {
        TA_BWD(8)
        TA_BWD(16)
        TA_BWD(32)
        TA_BWD(64)
        default:
            return cudaErrorInvalidValue;
    }
#undef TA_BWD
}

}  // namespace ta
