// tc_dev.cuh -- device helpers shared by the tensor-core compositor (composite.cu) and its backward
// pass (backward.cu): packed fp32x2 arithmetic, exp_det2, per-entry lane masks and culling of an 8x8
// pixel block, ldmatrix / mma.sync / cp.async wrappers (sm_100a).
#pragma once
#include <cuda_fp16.h>
#include "common.cuh"

namespace ta {

// Packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2): each component is one IEEE fp32
// operation rounded to nearest -- the same result as the scalar __f*_rn sequence, two pixels per
// instruction.
typedef unsigned long long u64x;
__device__ __forceinline__ u64x pk2(float2 a) { return *reinterpret_cast<const u64x*>(&a); }
__device__ __forceinline__ float2 up2(u64x a) { return *reinterpret_cast<const float2*>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    u64x r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return up2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    u64x r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return up2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    u64x r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return up2(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    u64x r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return up2(r);
}
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }

// exp_det (R13) of two arguments at once; identical per component to exp_det() for
// x >= -80 (the only arguments whose results are used: x = -q/2 with q <= q_max).
__device__ __forceinline__ float2 exp_det2(float2 x) {
    // k = the integer nearest (ties to even) to the exact product x*log2e, with one rounding:
    // fma(x, log2e, 1.5*2^23) lands on that integer (|x*log2e| < 2^22), the difference recovers it as
    // a float and the low mantissa bits hold it as an integer.  (Written as one fma on purpose: ptxas
    // contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2, so a separate product is not expressible.)
    constexpr float kMagic = 12582912.0f;                  // 1.5 * 2^23
    const float2 t = fma2(x, bc2(1.44269502162933349609375f), bc2(kMagic));
    const float2 k = sub2(t, bc2(kMagic));
    const float2 nk = make_float2(-k.x, -k.y);
    const float2 r = fma2(nk, bc2(0.693147182464599609375f), x);
    float2 p = bc2(1.3814548728987575e-3f);
    p = fma2(p, r, bc2(8.36869515478611e-3f));
    p = fma2(p, r, bc2(4.166838899254799e-2f));
    p = fma2(p, r, bc2(1.666652113199234e-1f));
    p = fma2(p, r, bc2(4.999999403953552e-1f));
    p = fma2(p, r, bc2(1.0f));
    p = fma2(p, r, bc2(1.0f));
    // p * 2^k as an exponent add on p's bits (integer pipe instead of an FMUL2 on the busy FMA pipe):
    // the same value as the multiply whenever the product is a normal number, i.e. for x >= -80 as
    // above (p in [0.7, 1.42], k >= -116); other lanes' values are never used
    const int kx = __float_as_int(t.x) - 0x4b400000, ky = __float_as_int(t.y) - 0x4b400000;
    return make_float2(__int_as_float(__float_as_int(p.x) + (kx << 23)), __int_as_float(__float_as_int(p.y) + (ky << 23)));
}

// exp of the staged argument x (= -q/2) for two values: the fixed sequence exp_det (R13,
// bit-identical to the oracle) or, for the opt-in fast mode (ta_raster_params.exact_exp = 0), the SFU:
// ex2.approx(x * log2 e) -- a few ulp from exp, so alpha' and, rarely, a stop decision may differ.
template <bool kFast>
__device__ __forceinline__ float2 exp2v(float2 x) {
    if constexpr (kFast) {
        const float2 y = mul2(x, bc2(1.44269504088896341f));
        float a, b;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(y.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(y.y));
        return make_float2(a, b);
    } else {
        return exp_det2(x);
    }
}

// Lanes of an 8x8 block (lane l: column l&7, row l>>3 (+4 for pixel B)) whose pixel lies inside the
// box [gx0,gx1]x[gy0,gy1]; computed once per staged entry instead of once per pixel.
__device__ __forceinline__ uint32_t box_lane_mask(int gx0, int gx1, int gy0, int gy1, int bx0, int ry) {
    const int cx0 = max(gx0 - bx0, 0), cx1 = min(gx1 - bx0, 7);
    const int ry0 = max(gy0 - ry, 0), ry1 = min(gy1 - ry, 3);
    if (cx0 > cx1 || ry0 > ry1) return 0u;
    const uint32_t col = (0xffu >> (7 - cx1)) & (0xffu << cx0);
    const int span = 8 * (ry1 - ry0 + 1);
    const uint32_t rows = (span >= 32 ? 0xffffffffu : ((1u << span) - 1u)) << (8 * ry0);
    return rows & (col * 0x01010101u);
}

// Both lane masks of an 8x8 block at once, branch-free: mA = lanes whose pixel A (rows by0 .. by0+3)
// lies in the box, mB = the same for pixel B (rows by0+4 .. by0+7).  The clamped ranges make an empty
// overlap give an empty 8-bit column / row mask; the 4 row bits of each half are spread to bytes by
// multiply-and-mask.  Equal to box_lane_mask(.., by0) / box_lane_mask(.., by0 + 4).
__device__ __forceinline__ void box_lane_masks(int gx0, int gx1, int gy0, int gy1, int bx0, int by0, uint32_t& mA,
                                               uint32_t& mB) {
    const int cx0 = min(max(gx0 - bx0, 0), 8), cx1 = max(min(gx1 - bx0, 7), -1);
    const int ry0 = min(max(gy0 - by0, 0), 8), ry1 = max(min(gy1 - by0, 7), -1);
    const uint32_t col = (0xffu >> (7 - cx1)) & (0xffu << cx0) & 0xffu;
    const uint32_t row = (0xffu >> (7 - ry1)) & (0xffu << ry0) & 0xffu;
    const uint32_t crep = col * 0x01010101u;
    const uint32_t ra = ((((row & 0xfu) * 0x00204081u) & 0x01010101u) * 0xffu);
    const uint32_t rb = ((((row >> 4) * 0x00204081u) & 0x01010101u) * 0xffu);
    mA = crep & ra;
    mB = crep & rb;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr) : "memory");
}
__device__ __forceinline__ void hmma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    // .cg: the staged feature rows bypass L1 (read once per warp; L1 is left to the splat records)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Bulk (non-tensor TMA) copy global -> shared of `bytes` (multiple of 16, both addresses 16-B aligned),
// completing as transaction bytes on the mbarrier at `bar`; and the mbarrier operations the fill uses.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra MBW_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
// The same wait with a suspend-time hint: a waiting warp sleeps (up to the hint) until the phase
// completes instead of re-issuing try_wait, leaving the issue slots to the SM's other warps.
__device__ __forceinline__ void mbar_wait_parity_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "MBS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra MBS_%=;\n}\n" ::"r"(bar), "r"(parity), "r"(1000000u) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Tensor memory as per-warp storage: 32 lanes x 16 consecutive 32-bit columns of the warp's lane
// quarter <-> 16 registers per thread (tcgen05.ld / st 32x32b.x16; asynchronous, fenced by the waits).
__device__ __forceinline__ void tm_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
          "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])),
          "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
          "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
          "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Conservative "may the ellipse q <= qlim reach the pixel rectangle [X0,X1] x [Y0,Y1]" test.  For a
// centre outside the rectangle the minimum of the convex q over it lies on an edge facing the centre
// (at a minimiser on x = X0 the gradient 2 C d has no y part, so d_x = (g_x / 2) Sigma_xx >= 0, i.e.
// mx <= X0; likewise for the other edges), so only those (at most one vertical and one horizontal)
// are evaluated, each at the clamped minimiser along it.  The approximate reciprocal only moves the
// evaluation point by ~1e-7 relative (q error second order); qlim carries a 1.6 % + 0.01 margin.
// Nearly degenerate conics (condition > 4096) are never culled (the per-pixel test decides).
__device__ __forceinline__ bool ellipse_may_touch2(float mx, float my, float ca, float cb2, float cc, float X0,
                                                   float X1, float Y0, float Y1, float qlim) {
    const float lx = X0 - mx, hx = X1 - mx, ly = Y0 - my, hy = Y1 - my;
    const bool vx = lx > 0.0f || hx < 0.0f, vy = ly > 0.0f || hy < 0.0f;
    if (!vx && !vy) return true;                       // centre inside
    const float cb = 0.5f * cb2;
    if (!(fmaf(-cb, cb, ca * cc) * 4096.0f > ca * cc)) return true;
    float best = 3.0e38f;
    if (vx) {
        const float dx = lx > 0.0f ? lx : hx;
        const float dy = fminf(fmaxf(-cb * dx * rcp_approx(cc), ly), hy);
        best = dx * (ca * dx + cb2 * dy) + cc * dy * dy;
    }
    if (vy) {
        const float ey = ly > 0.0f ? ly : hy;
        const float ex = fminf(fmaxf(-cb * ey * rcp_approx(ca), lx), hx);
        best = fminf(best, ex * (ca * ex + cb2 * ey) + cc * ey * ey);
    }
    return best <= qlim;
}
// The same test without branches (both edge minima always evaluated, then selected): the SIMT fill
// evaluates it for 32 list entries at once, where the branches of the form above diverge.
__device__ __forceinline__ bool ellipse_may_touch_bf(float mx, float my, float ca, float cb2, float cc, float X0,
                                                     float X1, float Y0, float Y1, float qlim) {
    const float lx = X0 - mx, hx = X1 - mx, ly = Y0 - my, hy = Y1 - my;
    const bool vx = lx > 0.0f || hx < 0.0f, vy = ly > 0.0f || hy < 0.0f;
    const float cb = 0.5f * cb2;
    const bool degenerate = !(fmaf(-cb, cb, ca * cc) * 4096.0f > ca * cc);
    const float dx = lx > 0.0f ? lx : hx;
    const float dy = fminf(fmaxf(-cb * dx * rcp_approx(cc), ly), hy);
    const float b1 = dx * (ca * dx + cb2 * dy) + cc * dy * dy;
    const float ey = ly > 0.0f ? ly : hy;
    const float ex = fminf(fmaxf(-cb * ey * rcp_approx(ca), lx), hx);
    const float b2 = ex * (ca * ex + cb2 * ey) + cc * ey * ey;
    const float best = fminf(vx ? b1 : 3.0e38f, vy ? b2 : 3.0e38f);
    return (!vx & !vy) | degenerate | (best <= qlim);
}

constexpr float kInf = __builtin_huge_valf();

// q = fma(fma(ca, dx, cb2*dy), dx, (cc*dy)*dy) for the lane's two pixels (normative a6 sequence)
__device__ __forceinline__ float2 quad_q(const float4 G, float cc, float pxf, float2 py2) {
    const float dx = fsub(pxf, G.x);
    const float2 dy = sub2(py2, bc2(G.y));
    const float2 t1 = mul2(bc2(G.w), dy);
    const float2 t2 = fma2(bc2(G.z), bc2(dx), t1);
    const float2 t4 = mul2(mul2(bc2(cc), dy), dy);
    return fma2(t2, bc2(dx), t4);
}

// One compositing step of the normative a6 recurrence for the lane's two pixels, in the staged
// scaling: q = q' = -q/2, a = 2^11 alpha', mA / mB = the entry's box lane masks (a pixel takes part
// only while its bit is also set in actA / actB); qlo = -q_max/2, alo = 2^11 alpha_min.  Both scalings are exact (powers of two, no
// subnormals on the used range), so every decision and T are those of the normative sequence:
// fma(a, -2^-11, 1) = fl(1 - alpha').  Returns the weight 2^11 alpha' T of each pixel (0 if it does
// not composite this entry) and advances T / the active bits.
template <bool kCounts>
__device__ __forceinline__ float2 tstep(float2 q, float2 a, uint32_t mA, uint32_t mB, float qlo, float alo, float teps,
                                        float2& T, uint32_t& actA, uint32_t& actB, int& ncA, int& ncB,
                                        unsigned long long* wk) {
    const float2 Tn = mul2(T, fma2(a, bc2(-1.0f / 2048.0f), bc2(1.0f)));
    const bool okA = (mA & actA) && q.x >= qlo && a.x >= alo, okB = (mB & actB) && q.y >= qlo && a.y >= alo;
    const bool inA = okA && Tn.x >= teps, inB = okB && Tn.y >= teps;
    if (okA && !inA) actA = 0u;           // T would drop below t_eps: stop before this Gaussian (R10)
    if (okB && !inB) actB = 0u;
    const float2 ws = mul2(a, T);
    const float2 w = make_float2(inA ? ws.x : 0.0f, inB ? ws.y : 0.0f);
    T = make_float2(inA ? Tn.x : T.x, inB ? Tn.y : T.y);
    if (kCounts) {
        wk[4] += __any_sync(0xffffffffu, inA || inB) ? 1 : 0;
        wk[5] += __popc(__ballot_sync(0xffffffffu, inA)) + __popc(__ballot_sync(0xffffffffu, inB));
        ncA += inA ? 1 : 0;
        ncB += inB ? 1 : 0;
    }
    return w;
}

}  // namespace ta
