// backward.cu -- SURVEY 8(f) NEXT #4: backward pass of the compositing step (sm_100a).
//
// Gradients of L = sum_p G_F(p) . F(p) + G_A(p) A(p) with respect to each Gaussian's 2D splat
// parameters (mean2, conic (ca, cb2, cc), alpha) and feature row, for the a6 forward of PAPER.md
// l.386-387 (the differentiable rasterizer of [kerbl20233d]); reading R25 (decisions held
// fixed, no gradient through a binding alpha clamp).  It reuses the splat records and the per-tile
// lists of the preceding ta_rasterize on the same context.
// Two kernels: k_composite_bwd_tc<C> (fp16-stored features, C in {16, 32, 64}; tensor cores, see the
// section comment below) and the plain k_composite_bwd (fp32-stored features and C = 8):
// one CTA per tile (16 x 16 or 8 x 8 pixels), one pixel per thread; the tile list is staged 256 entries at a time in
// shared memory (record + fp32 feature row).  Pass 1 replays the forward per pixel (the same fp32
// decision sequence as the forward kernels, so the composited set is identical) and accumulates
// S = sum w_j g_j (g_j = G_F . f_j) and T_end; pass 2 replays it again and forms every composited
// entry's per-pixel terms: dL/dalpha'_j = T_j g_j - (S - sum_{k<=j} w_k g_k)/(1 - alpha'_j)
// + G_A T_end/(1 - alpha'_j), chained to alpha, q, conic and mean2, and w_j G_F for the features.
// Per entry the 32 pixels of a warp are summed with shuffles and one lane adds them to the global
// gradient arrays (fp32 atomics: the summation order over warps is not fixed).
#include <algorithm>
#include <type_traits>
#include <cuda_bf16.h>
#include "common.cuh"
#include "internal.h"
#include "tc_dev.cuh"

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
    const int ts = cg.ts, TS = 1 << ts;               // tile side: 16 (256 threads) or 8 (64 threads)
    const int px = (txi << ts) + (int)(threadIdx.x & (TS - 1)), py = (tyi << ts) + (int)(threadIdx.x >> ts);
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

    // warp strip: threads 32w .. 32w+31 = pixel rows (32 / TS) w .. (32 / TS)(w + 1) - 1 of the tile, all TS columns
    const int rows = 32 >> ts;
    const int sy0 = (tyi << ts) + rows * (int)(threadIdx.x >> 5), sx0 = txi << ts;
    auto strip_hit = [&](uint32_t k) -> bool {
        const float4 Hh = s_h[k];
        const uint32_t bx = __float_as_uint(Hh.z), by = __float_as_uint(Hh.w);
        return (int)(bx & 0xffff) <= sx0 + TS - 1 && (int)(bx >> 16) >= sx0 && (int)(by & 0xffff) <= sy0 + rows - 1 &&
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

// ============================================================================ tensor-core variant
// k_composite_bwd_tc<C> (fp16-stored features, C in {16, 32, 64}): the forward compositor's layout --
// persistent warps over 8x8 blocks, lane l owning the pixels (l&7, l>>3) and (l&7, (l>>3)+4), entries
// culled against the block's still-active pixels and staged 16 at a time -- walked twice per block.
// The three per-entry contractions run on the tensor cores (mma.sync m16n8k16, fp32 accumulate):
//   g[p][j]      = G_F(p) . f_j          G[64 px x 16] = GF[64 x C] . f^T       (fp16 hi/lo GF, scaled)
//   dL/df_j      = sum_p w_pj G_F(p)     D[16 x C]     = W^T[16 x 64] . GF      (fp16 hi/lo both)
//   moments_j    = sum_p da_pj u(p)      M[16 x 8]     = DA^T[16 x 64] . U      (bf16 hi/lo, U exact)
// with da = dL/dalpha (per pixel) and u(p) = (1, x, y, x^2, xy, y^2) in block-local pixel
// coordinates.  dL/dq = -alpha_j / 2 * da (the same factor e links both), so the centre and conic
// gradients sum_p dq (dx, dy, dx^2, dx dy, dy^2) follow from the moments by expanding dx = x - mx'.
// Pass 1 replays the decisions (the forward's fp32 sequence) for S = sum_j w_j g_j and T_end; pass 2
// forms dL/dalpha'_j (R25) per pixel and entry, stages w, dq, dalpha in shared memory and reduces them
// over the 64 pixels with the MMAs above; one lane per entry adds the sums to the gradient arrays
// (fp32 atomics).  GF is scaled per block by a power of two (max |GF| -> 2^14) so its fp16 hi/lo
// split keeps ~22 bits; every result is unscaled exactly.

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void bmma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }
__device__ __forceinline__ uint32_t b2u(__nv_bfloat162 h) { return *reinterpret_cast<const uint32_t*>(&h); }

constexpr int kBwdBuf = 16;          // entries staged per round (one MMA k- or n-extent)

template <int C>
struct BwdBuf {
    static constexpr int PH = (((C + 8) / 8) & 1) ? C + 8 : C + 16;   // fp16 row pitch: odd number of 16-B chunks
    static constexpr int WP = 36;                                     // words per [entry][pixel'] row (144 B)
    float4 g[kBwdBuf];                 // mx, my, ca, cb2
    float4 h[kBwdBuf];                 // cc, alpha, box lane mask (pixel A), (pixel B)
    uint32_t id[kBwdBuf];              // array index
    __half f[kBwdBuf][PH];             // staged fp16 feature rows
    __half gf[2][64][PH];              // scaled GF, fp16 hi / lo, row p' = 2 lane + (0: pixel A, 1: pixel B)
    uint32_t w[2][kBwdBuf][WP];        // fp16 hi / lo of 2^11 w, word = lane: (pixel A, pixel B)
    union {
        float2 G[kBwdBuf][32];         // scaled g of (entry, lane): (pixel A, pixel B), read into registers
        uint32_t da[2][kBwdBuf][WP];   // then: bf16 hi / lo of dL/dalpha, word = lane: (pixel A, pixel B)
    };
    float mom[kBwdBuf][8];             // per entry: sum da (1, x, y, xx, xy, yy)
};

template <int C>
__global__ void __launch_bounds__(32) k_composite_bwd_tc(const uint4* __restrict__ rec, const __half* __restrict__ feat,
                                                         const uint32_t* __restrict__ tlist, const uint2* __restrict__ trng,
                                                         const uint32_t* __restrict__ order, CompositeGeom cg, RasterConsts rc,
                                                         CallState* __restrict__ cs, uint64_t list_cap,
                                                         const float* __restrict__ GF, const float* __restrict__ GA,
                                                         float* __restrict__ d_mean2, float* __restrict__ d_conic,
                                                         float* __restrict__ d_alpha, float* __restrict__ d_feat) {
    constexpr int PH = BwdBuf<C>::PH, WP = BwdBuf<C>::WP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdBuf<C>& bf = *reinterpret_cast<BwdBuf<C>*>(smem_raw);
    const uint32_t lane = lane_id();
    const int li = (int)lane, gq = li >> 2, tq = li & 3;
    const uint32_t lt = lanemask_lt();
    const uint32_t n = cs->n;
    const int W = cg.W, H = cg.H;
    const float qmax = rc.q_max, amax = rc.alpha_max, amin = rc.alpha_min, teps = rc.t_eps;
    const float qlim = qmax * 1.015625f + 0.01f;

    // U fragments (B operand of the moment MMA, constant): element k of k-step ks is pixel p' = 16 ks + k
    uint32_t ub[4][2];
#pragma unroll
    for (int ks = 0; ks < 4; ks++)
#pragma unroll
        for (int hf = 0; hf < 2; hf++) {
            const int l2 = 8 * ks + tq + 4 * hf;             // lane of pixels p' = 2 l2 (A), 2 l2 + 1 (B)
            const float x = (float)(l2 & 7), yA = (float)(l2 >> 3), yB = yA + 4.0f;
            auto u = [&](float y) {
                switch (gq) {
                    case 0: return 1.0f;
                    case 1: return x;
                    case 2: return y;
                    case 3: return x * x;
                    case 4: return x * y;
                    case 5: return y * y;
                    default: return 0.0f;
                }
            };
            ub[ks][hf] = b2u(__floats2bfloat162_rn(u(yA), u(yB)));
        }
    // ldmatrix lane addresses
    const uint32_t gf_a = smem_u32(&bf.gf[0][(li & 7) + 8 * ((li >> 3) & 1)][8 * (li >> 4)]);     // A: GF rows, + 16 mt rows, + 16 ks cols
    const uint32_t f_b = smem_u32(&bf.f[(li & 7) + 8 * (li >> 4)][8 * ((li >> 3) & 1)]);          // B: f rows (entries), + 16 ks cols
    const uint32_t gf_bt = smem_u32(&bf.gf[0][(li & 7) + 8 * ((li >> 3) & 1)][8 * (li >> 4)]);    // B (trans): GF rows p', + 16 ks rows, + 16 np cols
    const uint32_t w_a = smem_u32(&bf.w[0][(li & 7) + 8 * ((li >> 3) & 1)][4 * (li >> 4)]);        // A: W rows (entries), + 8 ks words
    const uint32_t da_a = smem_u32(&bf.da[0][(li & 7) + 8 * ((li >> 3) & 1)][4 * (li >> 4)]);
    constexpr uint32_t kGfLo = 64 * PH * 2, kWLo = kBwdBuf * WP * 4;

    uint32_t* const wq = &cs->scan_counter[7];
    const bool t8 = cg.ts == 3;
    const uint32_t nblk = (t8 ? 1u : 4u) * (uint32_t)(cg.TX * cg.TY);
    for (;;) {
        uint32_t blk = 0;
        if (lane == 0) blk = atomicAdd(wq, 1u);
        blk = __shfl_sync(0xffffffffu, blk, 0);
        if (blk >= nblk) break;
        const int tile = (int)order[t8 ? blk : blk >> 2];
        const uint32_t qd = t8 ? 0u : blk & 3u;
        const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
        const uint2 tr = trng[tile];
        const uint32_t cstart = tr.x;
        uint32_t cend = tr.x + tr.y;
        if (cend > list_cap) cend = (uint32_t)list_cap;
        const int bx0 = (txi << cg.ts) + 8 * (int)(qd & 1), by0 = (tyi << cg.ts) + 8 * (int)(qd >> 1);
        const int px = bx0 + (li & 7), pyA = by0 + (li >> 3), pyB = pyA + 4;
        const float pxf = (float)px;
        const float2 py2 = make_float2((float)pyA, (float)pyB);
        const bool inA = px < W && pyA < H, inB = px < W && pyB < H;

        // ---- GF of the block, scaled by gsc = 2^(14 - e) (max |GF| = 2^e ... 2^(e+1)), fp16 hi / lo
        float mx_abs = 0.0f;
        {
            const float* rA = GF + ((size_t)pyA * W + px) * C;
            const float* rB = GF + ((size_t)pyB * W + px) * C;
#pragma unroll 4
            for (int c = 0; c < C; c += 4) {
                if (inA) {
                    const float4 v = *reinterpret_cast<const float4*>(rA + c);
                    mx_abs = fmaxf(mx_abs, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                }
                if (inB) {
                    const float4 v = *reinterpret_cast<const float4*>(rB + c);
                    mx_abs = fmaxf(mx_abs, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                }
            }
        }
        mx_abs = __reduce_max_sync(0xffffffffu, __float_as_uint(mx_abs)) == 0u ? 0.0f
                 : __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mx_abs)));
        const int ex = mx_abs > 0.0f ? (int)((__float_as_uint(mx_abs) >> 23) & 255u) - 127 : 0;
        const int sh = min(max(14 - ex, -100), 100);
        const float gsc = ldexpf(1.0f, sh), igsc = ldexpf(1.0f, -sh);
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            const bool ok = hh ? inB : inA;
            const float* r = GF + ((size_t)(hh ? pyB : pyA) * W + px) * C;
            __half* hi = &bf.gf[0][2 * li + hh][0];
            __half* lo = &bf.gf[1][2 * li + hh][0];
#pragma unroll 4
            for (int c = 0; c < C; c += 2) {
                const float2 v = ok ? *reinterpret_cast<const float2*>(r + c) : make_float2(0.0f, 0.0f);
                const float2 sv = make_float2(v.x * gsc, v.y * gsc);
                const __half2 h2 = __floats2half2_rn(sv.x, sv.y);
                const float2 hf = __half22float2(h2);
                *reinterpret_cast<__half2*>(hi + c) = h2;
                *reinterpret_cast<__half2*>(lo + c) = __floats2half2_rn(sv.x - hf.x, sv.y - hf.y);
            }
        }
        const float2 ga2 = make_float2(inA ? GA[(size_t)pyA * W + px] * gsc : 0.0f,
                                       inB ? GA[(size_t)pyB * W + px] * gsc : 0.0f);
        __syncwarp();

        float2 S = make_float2(0.0f, 0.0f), Tend = make_float2(1.0f, 1.0f);
        for (int pass = 0; pass < 2; pass++) {
            float2 T = make_float2(1.0f, 1.0f), Sup = make_float2(0.0f, 0.0f);
            uint32_t actA = inA ? (1u << lane) : 0u, actB = inB ? (1u << lane) : 0u;
            uint32_t pos = cstart;
            uint32_t pf_pos = 0xffffffffu, pf = 0u;          // list index of entry pf_pos + lane, loaded ahead
            while (pos < cend && __any_sync(0xffffffffu, (actA | actB) != 0u)) {
                // culling rectangle = bounding box of the pixels still compositing
                const int lx0 = (actA | actB) ? px : 0x7fffffff, lx1 = (actA | actB) ? px : -1;
                const int ly0 = actA ? pyA : (actB ? pyB : 0x7fffffff), ly1 = actB ? pyB : (actA ? pyA : -1);
                const int ax0 = __reduce_min_sync(0xffffffffu, lx0), ax1 = __reduce_max_sync(0xffffffffu, lx1);
                const int ay0 = __reduce_min_sync(0xffffffffu, ly0), ay1 = __reduce_max_sync(0xffffffffu, ly1);
                const float X0 = (float)ax0, X1 = (float)ax1, Y0 = (float)ay0, Y1 = (float)ay1;
                // ---- fill: up to 16 entries in list order (32 list entries per round trip)
                int cnt = 0;
                while (cnt < kBwdBuf && pos < cend) {
                    const uint32_t e = pos + lane;
                    const uint32_t idx = pf_pos == pos ? pf : (e < cend ? tlist[e] : 0xffffffffu);
                    const uint32_t i = idx < n ? idx : 0u;
                    const uint4 r1 = rec[2 * i + 1], r0 = rec[2 * i];
                    pf_pos = pos + 32;
                    pf = pos + 32 + lane < cend ? tlist[pos + 32 + lane] : 0xffffffffu;
                    const int gx0 = (int)(r1.z & 0xffff), gx1 = (int)(r1.z >> 16);
                    const int gy0 = (int)(r1.w & 0xffff), gy1 = (int)(r1.w >> 16);
                    bool kp = (idx < n) & (gx0 <= ax1) & (gx1 >= ax0) & (gy0 <= ay1) & (gy1 >= ay0) &
                              ellipse_may_touch_bf(__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z),
                                                   __uint_as_float(r0.w), __uint_as_float(r1.x), X0, X1, Y0, Y1, qlim);
                    uint32_t bal = __ballot_sync(0xffffffffu, kp);
                    const int room = kBwdBuf - cnt;
                    const uint32_t rank = __popc(bal & lt);
                    uint32_t step = min(32u, cend - pos);
                    if (__popc(bal) > room) {
                        const uint32_t cut = __ballot_sync(0xffffffffu, kp && rank == (uint32_t)room);
                        const int cl = __ffs(cut) - 1;
                        bal &= (1u << cl) - 1u;
                        step = (uint32_t)cl;
                        kp = kp && li < cl;
                    }
                    if (kp) {
                        const int d = cnt + (int)rank;
                        bf.g[d] = make_float4(__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z),
                                              __uint_as_float(r0.w));
                        uint32_t mA, mB;
                        box_lane_masks(gx0, gx1, gy0, gy1, bx0, by0, mA, mB);
                        bf.h[d] = make_float4(__uint_as_float(r1.x), __uint_as_float(r1.y), __uint_as_float(mA),
                                              __uint_as_float(mB));
                        bf.id[d] = idx;
                        const char* src = reinterpret_cast<const char*>(feat + (size_t)idx * C);
                        const uint32_t dst = smem_u32(&bf.f[d][0]);
#pragma unroll
                        for (int c = 0; c < C * 2; c += 16) cp_async16(dst + c, src + c);
                    }
                    cnt += __popc(bal);
                    pos += step;
                }
                cp_async_wait_all();
                __syncwarp();
                if (cnt == 0) continue;
                // ---- g = GF . f^T on the tensor cores -> bf.G[entry][lane] (pixel A, pixel B)
#pragma unroll
                for (int mt = 0; mt < 4; mt++) {
                    float acc[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
#pragma unroll
                    for (int ks = 0; ks < C / 16; ks++) {
                        uint32_t ah[4], al[4], b[4];
                        const uint32_t aa = gf_a + (uint32_t)((16 * mt * PH + 16 * ks) * 2);
                        ldsm_x4(aa, ah[0], ah[1], ah[2], ah[3]);
                        ldsm_x4(aa + kGfLo, al[0], al[1], al[2], al[3]);
                        ldsm_x4(f_b + (uint32_t)(16 * ks * 2), b[0], b[1], b[2], b[3]);
                        hmma16816(acc[0], ah, b[0], b[1]);
                        hmma16816(acc[0], al, b[0], b[1]);
                        hmma16816(acc[1], ah, b[2], b[3]);
                        hmma16816(acc[1], al, b[2], b[3]);
                    }
                    // row r = 16 mt + gq (+8) is pixel p' = r: lane r >> 1, component r & 1
#pragma unroll
                    for (int nt = 0; nt < 2; nt++)
#pragma unroll
                        for (int e2 = 0; e2 < 4; e2++) {
                            const int r = 16 * mt + gq + 8 * (e2 >> 1), col = 8 * nt + 2 * tq + (e2 & 1);
                            reinterpret_cast<float*>(&bf.G[col][r >> 1])[r & 1] = acc[nt][e2];
                        }
                }
                __syncwarp();
                float2 gv[kBwdBuf];                        // this lane's g of the staged entries
#pragma unroll
                for (int j = 0; j < kBwdBuf; j++) gv[j] = bf.G[j][lane];
                __syncwarp();                              // bf.G is overwritten by bf.da below
                // ---- the recurrence (decisions = the forward's fp32 sequence).  Full chunks of 16 take a
                //      branch-free copy so the scheduler can overlap consecutive entries.
                auto recur = [&](auto full, auto second) {
                    constexpr bool kFull = decltype(full)::value, kP2 = decltype(second)::value;
#pragma unroll
                    for (int j = 0; j < kBwdBuf; j++) {
                        float2 w = make_float2(0.0f, 0.0f), dal = make_float2(0.0f, 0.0f);
                        if (kFull || j < cnt) {
                            const float4 G0 = bf.g[j], H0 = bf.h[j];
                            const float2 q = quad_q(G0, H0.x, pxf, py2);
                            const float2 qm = make_float2((__float_as_uint(H0.z) & actA) ? q.x : kInf,
                                                          (__float_as_uint(H0.w) & actB) ? q.y : kInf);
                            const float2 ee = exp_det2(mul2(bc2(-0.5f), q));
                            const float2 ae = mul2(bc2(H0.y), ee);
                            const float2 a = make_float2(fminf(amax, ae.x), fminf(amax, ae.y));
                            const float2 om = sub2(bc2(1.0f), a);
                            const float2 Tn = mul2(T, om);
                            const bool okA = qm.x <= qmax && a.x >= amin, okB = qm.y <= qmax && a.y >= amin;
                            const bool tA = okA && Tn.x >= teps, tB = okB && Tn.y >= teps;
                            if (okA && !tA) actA = 0u;
                            if (okB && !tB) actB = 0u;
                            const float2 gg = gv[j];
                            w = make_float2(tA ? fmul(a.x, T.x) : 0.0f, tB ? fmul(a.y, T.y) : 0.0f);
                            if (!kP2) {
                                S = make_float2(ffma(w.x, gg.x, S.x), ffma(w.y, gg.y, S.y));
                            } else {
                                Sup = make_float2(ffma(w.x, gg.x, Sup.x), ffma(w.y, gg.y, Sup.y));
                                // dL/dalpha' (R25) = T g - (S - Sup) / (1 - alpha') + G_A T_end / (1 - alpha'), per
                                // pixel, scaled by gsc like g and S; dL/dalpha = dL/dalpha' e unless clamped
                                const float2 num = sub2(mul2(ga2, Tend), sub2(S, Sup));
                                const float2 r = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                                const float2 dad = fma2(T, gg, mul2(num, r));
                                const float2 d = mul2(dad, ee);
                                dal = make_float2((tA && !(ae.x > amax)) ? d.x : 0.0f, (tB && !(ae.y > amax)) ? d.y : 0.0f);
                            }
                            T = make_float2(tA ? Tn.x : T.x, tB ? Tn.y : T.y);
                        }
                        if (kP2) {                         // rows j >= cnt are written as zeros
                            const float2 ws = mul2(w, bc2(2048.0f));
                            const __half2 wh = __floats2half2_rn(ws.x, ws.y);
                            const float2 whf = __half22float2(wh);
                            bf.w[0][j][li] = h2u(wh);
                            bf.w[1][j][li] = h2u(__floats2half2_rn(ws.x - whf.x, ws.y - whf.y));
                            const __nv_bfloat162 lh = __floats2bfloat162_rn(dal.x, dal.y);
                            const float2 lhf = __bfloat1622float2(lh);
                            bf.da[0][j][li] = b2u(lh);
                            bf.da[1][j][li] = b2u(__floats2bfloat162_rn(dal.x - lhf.x, dal.y - lhf.y));
                        }
                    }
                };
                using T_ = std::true_type;
                using F_ = std::false_type;
                if (pass == 0) {
                    if (cnt == kBwdBuf) recur(T_(), F_());
                    else recur(F_(), F_());
                } else {
                    if (cnt == kBwdBuf) recur(T_(), T_());
                    else recur(F_(), T_());
                }
                __syncwarp();
                if (pass == 0) continue;
                // ---- dL/df = W^T . GF: rows = entries, cols = channels
#pragma unroll
                for (int np = 0; np < C / 16; np++) {
                    float acc[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
#pragma unroll
                    for (int ks = 0; ks < 4; ks++) {
                        uint32_t ah[4], al[4], bh[4], bl[4];
                        ldsm_x4(w_a + (uint32_t)(32 * ks), ah[0], ah[1], ah[2], ah[3]);
                        ldsm_x4(w_a + (uint32_t)(32 * ks) + kWLo, al[0], al[1], al[2], al[3]);
                        const uint32_t bb = gf_bt + (uint32_t)((16 * ks * PH + 16 * np) * 2);
                        ldsm_x4_t(bb, bh[0], bh[1], bh[2], bh[3]);
                        ldsm_x4_t(bb + kGfLo, bl[0], bl[1], bl[2], bl[3]);
#pragma unroll
                        for (int nt = 0; nt < 2; nt++) {
                            hmma16816(acc[nt], ah, bh[2 * nt], bh[2 * nt + 1]);
                            hmma16816(acc[nt], ah, bl[2 * nt], bl[2 * nt + 1]);
                            hmma16816(acc[nt], al, bh[2 * nt], bh[2 * nt + 1]);
                        }
                    }
                    const float sc = igsc * (1.0f / 2048.0f);
#pragma unroll
                    for (int nt = 0; nt < 2; nt++)
#pragma unroll
                        for (int e2 = 0; e2 < 4; e2++) {
                            const int row = gq + 8 * (e2 >> 1), c = 16 * np + 8 * nt + 2 * tq + (e2 & 1);
                            if (row < cnt) atomicAdd(d_feat + (size_t)bf.id[row] * C + c, acc[nt][e2] * sc);
                        }
                }
                // ---- moments: DA^T . U
                {
                    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                    for (int ks = 0; ks < 4; ks++) {
                        uint32_t ah[4], al[4];
                        ldsm_x4(da_a + (uint32_t)(32 * ks), ah[0], ah[1], ah[2], ah[3]);
                        ldsm_x4(da_a + (uint32_t)(32 * ks) + kWLo, al[0], al[1], al[2], al[3]);
                        bmma16816(acc, ah, ub[ks][0], ub[ks][1]);
                        bmma16816(acc, al, ub[ks][0], ub[ks][1]);
                    }
#pragma unroll
                    for (int e2 = 0; e2 < 4; e2++) bf.mom[gq + 8 * (e2 >> 1)][2 * tq + (e2 & 1)] = acc[e2];
                }
                __syncwarp();
                if (li < cnt) {                            // one lane per entry: the scalar gradients
                    const float4 G0 = bf.g[li];
                    const float cc = bf.h[li].x;
                    const float* m = bf.mom[li];
                    const float mxl = G0.x - (float)bx0, myl = G0.y - (float)by0;
                    const float M0 = m[0], Mx = m[1], My = m[2], Mxx = m[3], Mxy = m[4], Myy = m[5];
                    const float k = -0.5f * bf.h[li].y * igsc;   // dL/dq = -alpha / 2 * dL/dalpha
                    const float Sdx = k * (Mx - mxl * M0), Sdy = k * (My - myl * M0);
                    const float Sdxx = k * (Mxx - 2.0f * mxl * Mx + mxl * mxl * M0);
                    const float Sdxy = k * (Mxy - mxl * My - myl * Mx + mxl * myl * M0);
                    const float Sdyy = k * (Myy - 2.0f * myl * My + myl * myl * M0);
                    const uint32_t gi = bf.id[li];
                    atomicAdd(d_alpha + gi, M0 * igsc);
                    atomicAdd(d_conic + 3 * (size_t)gi + 0, Sdxx);
                    atomicAdd(d_conic + 3 * (size_t)gi + 1, Sdxy);
                    atomicAdd(d_conic + 3 * (size_t)gi + 2, Sdyy);
                    atomicAdd(d_mean2 + 2 * (size_t)gi + 0, -(2.0f * G0.z * Sdx + G0.w * Sdy));
                    atomicAdd(d_mean2 + 2 * (size_t)gi + 1, -(G0.w * Sdx + 2.0f * cc * Sdy));
                }
                __syncwarp();
            }
            if (pass == 0) Tend = T;
        }
    }
}

template <int C>
static cudaError_t launch_bwd_tc(int tiles, int resident, const uint4* rec, const void* feat, const uint32_t* tlist, const uint2* trng,
                                 const uint32_t* order, CompositeGeom cg, RasterConsts rc, CallState* cs,
                                 uint64_t list_cap, const float* GF, const float* GA, float* d_mean2, float* d_conic,
                                 float* d_alpha, float* d_feat, cudaStream_t st) {
    const size_t smem = sizeof(BwdBuf<C>);
    cudaError_t e = cudaMemsetAsync(&cs->scan_counter[7], 0, 4, st);
    if (e != cudaSuccess) return e;
    k_composite_bwd_tc<C><<<std::min((cg.ts == 3 ? 1 : 4) * tiles, resident), 32, smem, st>>>(
        rec, static_cast<const __half*>(feat), tlist, trng, order, cg, rc, cs, list_cap, GF, GA, d_mean2, d_conic,
        d_alpha, d_feat);
    return cudaGetLastError();
}

// Per-device preparation (ta_context_create, the context's device current): shared-memory opt-ins of
// the backward kernels and the co-resident grid of the persistent tensor-core backward per C.
template <int C>
static cudaError_t prepare_bwd_tc(int num_sms, int* resident) {
    const size_t smem = sizeof(BwdBuf<C>);
    cudaError_t e = cudaFuncSetAttribute(k_composite_bwd_tc<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_composite_bwd_tc<C>, 32, smem))) return e;
    *resident = std::max(1, num_sms * std::max(1, per_sm));
    return cudaSuccess;
}

cudaError_t prepare_composite_bwd(int num_sms, int resident[4]) {
    const int smem = (int)((size_t)kBwdBatch * (16 + 16 + 4 + 4 * (size_t)64));
    cudaError_t e;
#define TA_BWD_ATTR(CC)                                                                                                  \
    if ((e = cudaFuncSetAttribute(k_composite_bwd<CC, __half>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) ||  \
        (e = cudaFuncSetAttribute(k_composite_bwd<CC, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)))      \
        return e;
    TA_BWD_ATTR(8) TA_BWD_ATTR(16) TA_BWD_ATTR(32) TA_BWD_ATTR(64)
#undef TA_BWD_ATTR
    resident[0] = 1;
    if ((e = prepare_bwd_tc<16>(num_sms, &resident[1])) || (e = prepare_bwd_tc<32>(num_sms, &resident[2])) ||
        (e = prepare_bwd_tc<64>(num_sms, &resident[3])))
        return e;
    return cudaSuccess;
}

cudaError_t launch_composite_bwd(int C, int fbytes, int tiles, const int* resident, bool simt, const uint4* rec, const void* feat, const uint32_t* tlist,
                                 const uint2* trng, const uint32_t* order, CompositeGeom cg, RasterConsts rc,
                                 CallState* cs, uint64_t list_cap, const float* GF, const float* GA, float* d_mean2,
                                 float* d_conic, float* d_alpha, float* d_feat, cudaStream_t st) {
    const size_t smem = (size_t)kBwdBatch * (16 + 16 + 4 + 4 * (size_t)C);
    k_bwd_zero<<<1184, 256, 0, st>>>(cs, C, d_mean2, d_conic, d_alpha, d_feat);
    if (fbytes == 2 && tiles > 0 && !simt) {
        switch (C) {
            case 16: return launch_bwd_tc<16>(tiles, resident[1], rec, feat, tlist, trng, order, cg, rc, cs, list_cap, GF, GA, d_mean2,
                                              d_conic, d_alpha, d_feat, st);
            case 32: return launch_bwd_tc<32>(tiles, resident[2], rec, feat, tlist, trng, order, cg, rc, cs, list_cap, GF, GA, d_mean2,
                                              d_conic, d_alpha, d_feat, st);
            case 64: return launch_bwd_tc<64>(tiles, resident[3], rec, feat, tlist, trng, order, cg, rc, cs, list_cap, GF, GA, d_mean2,
                                              d_conic, d_alpha, d_feat, st);
            default: break;
        }
    }
    const int bthreads = 1 << (2 * cg.ts);       // one thread per pixel of the tile
#define TA_BWD(CC)                                                                                                      \
    case CC: {                                                                                                          \
        if (fbytes == 2) {                                                                                              \
            k_composite_bwd<CC, __half><<<tiles, bthreads, smem, st>>>(rec, static_cast<const __half*>(feat), tlist, \
                                                                          trng, cg, rc, cs, list_cap, GF, GA, d_mean2,  \
                                                                          d_conic, d_alpha, d_feat);                    \
        } else {                                                                                                        \
            k_composite_bwd<CC, float><<<tiles, bthreads, smem, st>>>(rec, static_cast<const float*>(feat), tlist,   \
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
