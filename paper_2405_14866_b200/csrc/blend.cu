// blend.cu -- SURVEY 8(f) NEXT #1: occlusion-aware input-view blending (sm_100a).
//
// PAPER.md l.420-444, Eqs. 6-10: every pixel of the fused depth z_fused (ta_zbuffer of all input
// views into the novel camera) is lifted (Pi_novel^-1), projected into each input view (Eq. 6),
// colour and depth are sampled bilinearly there (Eq. 7), weighted by
// w_i = M_i * Occ * cos<r, n_i> / ||x_i^cam|| (Eqs. 8-9) and normalised (Eq. 10).  DESIGN.md R24
// fixes the open points (tap rule, edge mask, appearance-consistency mask, finite-difference normals,
// cosine clamp, holes).
// One thread per novel pixel; views in index order; every step is the fp32 sequence of the
// oracle's tao_blend written with explicit __f*_rn intrinsics (no contraction), so the result
// is bit-identical to it.  The input maps are gathered through the read-only path (L1/L2): the
// four 1024^2 views (disparity, mask, RGB: 71 MB) stay L2-resident while a view is blended.
#include "common.cuh"
#include "internal.h"

namespace ta {

__device__ __forceinline__ bool bv_depth(const BlendView& v, int x, int y, float d_min, float* z) {
    if (x < 0 || y < 0 || x >= v.W || y >= v.H) return false;
    const size_t i = (size_t)y * v.W + x;
    if (v.mask && __ldg(v.mask + i) == 0) return false;
    const float d = __ldg(v.disp + i);
    if (!(isfinite(d) && d > d_min)) return false;
    *z = fdiv(v.fxB, d);
    return true;
}

__device__ __forceinline__ float lerp_rn(float a, float b, float t) { return ffma(t, fsub(b, a), a); }

__device__ __forceinline__ float lift_x(float px, float c, float f, float z) { return fmul(fdiv(fsub(px, c), f), z); }

__global__ void __launch_bounds__(256) k_blend(BlendTable bt, TargetCam cam, const float* __restrict__ zf,
                                               float* __restrict__ rgb, float* __restrict__ wsum) {
    const uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t npix = (uint32_t)cam.H * (uint32_t)cam.W;
    if (pix >= npix) return;
    const int v = (int)(pix / (uint32_t)cam.W), u = (int)(pix - (uint32_t)v * cam.W);
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f, ws = 0.0f;
    float sw[kMaxViews], sc[kMaxViews][3];              // pass 1: every contributing view's w_i, c_i
    int ns = 0;
    const float z = zf[pix];
    if (z > 0.0f) {
        const float* R = cam.R;
        const float* t = cam.t;
        // Eq. 6: Pi_novel^-1 (u, v, z_fused); ray from the novel centre C = R^T (0 - t)
        const float q0 = fsub(lift_x((float)u, cam.cx, cam.fx, z), t[0]);
        const float q1 = fsub(lift_x((float)v, cam.cy, cam.fy, z), t[1]);
        const float q2 = fsub(z, t[2]);
        const float w0 = dot3(R[0], R[3], R[6], q0, q1, q2);
        const float w1 = dot3(R[1], R[4], R[7], q0, q1, q2);
        const float w2 = dot3(R[2], R[5], R[8], q0, q1, q2);
        const float c0 = dot3(R[0], R[3], R[6], -t[0], -t[1], -t[2]);
        const float c1 = dot3(R[1], R[4], R[7], -t[0], -t[1], -t[2]);
        const float c2 = dot3(R[2], R[5], R[8], -t[0], -t[1], -t[2]);
        float r0 = fsub(w0, c0), r1 = fsub(w1, c1), r2 = fsub(w2, c2);
        const float rl = fsqrt(dot3(r0, r1, r2, r0, r1, r2));
        r0 = fdiv(r0, rl); r1 = fdiv(r1, rl); r2 = fdiv(r2, rl);
#pragma unroll 1
        for (int i = 0; i < bt.V; i++) {
            const BlendView& bv = bt.v[i];
            const float* Ri = bv.R;
            const float X = fadd(dot3(Ri[0], Ri[1], Ri[2], w0, w1, w2), bv.t[0]);
            const float Y = fadd(dot3(Ri[3], Ri[4], Ri[5], w0, w1, w2), bv.t[1]);
            const float Z = fadd(dot3(Ri[6], Ri[7], Ri[8], w0, w1, w2), bv.t[2]);
            if (!(Z > bt.z_near)) continue;
            const float us = ffma(bv.fx, fdiv(X, Z), bv.cx);
            const float vs = ffma(bv.fy, fdiv(Y, Z), bv.cy);
            if (!(us >= 0.0f && us <= (float)(bv.W - 1) && vs >= 0.0f && vs <= (float)(bv.H - 1))) continue;
            // Eq. 7: bilinear taps (R24)
            int x0 = (int)floorf(us), y0 = (int)floorf(vs);
            if (x0 > bv.W - 2) x0 = bv.W >= 2 ? bv.W - 2 : 0;
            if (y0 > bv.H - 2) y0 = bv.H >= 2 ? bv.H - 2 : 0;
            const int x1 = x0 + 1 < bv.W ? x0 + 1 : x0, y1 = y0 + 1 < bv.H ? y0 + 1 : y0;
            const float ax = fsub(us, (float)x0), ay = fsub(vs, (float)y0);
            float z00, z10, z01, z11;
            if (!bv_depth(bv, x0, y0, bt.d_min, &z00) || !bv_depth(bv, x1, y0, bt.d_min, &z10) ||
                !bv_depth(bv, x0, y1, bt.d_min, &z01) || !bv_depth(bv, x1, y1, bt.d_min, &z11))
                continue;
            const float zs = lerp_rn(lerp_rn(z00, z10, ax), lerp_rn(z01, z11, ax), ay);
            // Eq. 9: occlusion (SDF) check
            if (!(fabsf(fsub(Z, zs)) < bt.delta)) continue;
            // M_i: edge mask and a valid normal at the nearest pixel
            const int px = (int)rintf(us), py = (int)rintf(vs);
            float zc, zl, zr, zu, zd;
            if (!bv_depth(bv, px, py, bt.d_min, &zc) || !bv_depth(bv, px - 1, py, bt.d_min, &zl) ||
                !bv_depth(bv, px + 1, py, bt.d_min, &zr) || !bv_depth(bv, px, py - 1, bt.d_min, &zu) ||
                !bv_depth(bv, px, py + 1, bt.d_min, &zd))
                continue;
            if (fmul(fmaxf(fabsf(fsub(zr, zl)), fabsf(fsub(zd, zu))), 0.5f) > bt.edge_tau) continue;
            const float pxf = (float)px, pyf = (float)py;
            const float lx = lift_x(fsub(pxf, 1.0f), bv.cx, bv.fx, zl), ly = lift_x(pyf, bv.cy, bv.fy, zl);
            const float rx = lift_x(fadd(pxf, 1.0f), bv.cx, bv.fx, zr), ry = lift_x(pyf, bv.cy, bv.fy, zr);
            const float ux = lift_x(pxf, bv.cx, bv.fx, zu), uy = lift_x(fsub(pyf, 1.0f), bv.cy, bv.fy, zu);
            const float dx = lift_x(pxf, bv.cx, bv.fx, zd), dy = lift_x(fadd(pyf, 1.0f), bv.cy, bv.fy, zd);
            const float tx0 = fsub(rx, lx), tx1 = fsub(ry, ly), tx2 = fsub(zr, zl);
            const float ty0 = fsub(dx, ux), ty1 = fsub(dy, uy), ty2 = fsub(zd, zu);
            float n0 = ffma(tx1, ty2, -fmul(tx2, ty1));
            float n1 = ffma(tx2, ty0, -fmul(tx0, ty2));
            float n2 = ffma(tx0, ty1, -fmul(tx1, ty0));
            const float nl = fsqrt(dot3(n0, n1, n2, n0, n1, n2));
            if (!(nl > 0.0f)) continue;
            n0 = fdiv(n0, nl); n1 = fdiv(n1, nl); n2 = fdiv(n2, nl);
            const float pcx = lift_x(pxf, bv.cx, bv.fx, zc), pcy = lift_x(pyf, bv.cy, bv.fy, zc);
            if (dot3(n0, n1, n2, pcx, pcy, zc) > 0.0f) { n0 = -n0; n1 = -n1; n2 = -n2; }
            const float m0 = dot3(Ri[0], Ri[3], Ri[6], n0, n1, n2);
            const float m1 = dot3(Ri[1], Ri[4], Ri[7], n0, n1, n2);
            const float m2 = dot3(Ri[2], Ri[5], Ri[8], n0, n1, n2);
            // Eq. 8
            const float cs = -dot3(r0, r1, r2, m0, m1, m2);
            if (!(cs > 0.0f)) continue;
            const float dist = fsqrt(dot3(X, Y, Z, X, Y, Z));
            const float w = fdiv(cs, dist);
            const float* c00 = bv.color + ((size_t)y0 * bv.W + x0) * 3;
            const float* c10 = bv.color + ((size_t)y0 * bv.W + x1) * 3;
            const float* c01 = bv.color + ((size_t)y1 * bv.W + x0) * 3;
            const float* c11 = bv.color + ((size_t)y1 * bv.W + x1) * 3;
#pragma unroll
            for (int k = 0; k < 3; k++)
                sc[ns][k] = lerp_rn(lerp_rn(__ldg(c00 + k), __ldg(c10 + k), ax), lerp_rn(__ldg(c01 + k), __ldg(c11 + k), ax), ay);
            sw[ns++] = w;
        }
        // M_i's appearance-consistency mask (R24): m = the weighted median sample (medoid,
        // the c_i minimising sum_j w_j |c_j - c_i|, ties to the lower view), keep |c_i - m|^2 <= tau_c^2
        float m0 = 0.0f, m1 = 0.0f, m2 = 0.0f;
        if (bt.tau_c > 0.0f && ns > 0) {
            float best = __int_as_float(0x7f800000);
            int bi = 0;
#pragma unroll 1
            for (int i = 0; i < ns; i++) {
                float cost = 0.0f;
#pragma unroll 1
                for (int j = 0; j < ns; j++) {
                    const float e0 = fsub(sc[j][0], sc[i][0]), e1 = fsub(sc[j][1], sc[i][1]), e2 = fsub(sc[j][2], sc[i][2]);
                    cost = ffma(sw[j], fsqrt(dot3(e0, e1, e2, e0, e1, e2)), cost);
                }
                if (cost < best) { best = cost; bi = i; }
            }
            m0 = sc[bi][0]; m1 = sc[bi][1]; m2 = sc[bi][2];
        }
        const float tau2 = fmul(bt.tau_c, bt.tau_c);
        // pass 2: Eq. 10 sums over the consistent samples, in view order
#pragma unroll 1
        for (int i = 0; i < ns; i++) {
            if (bt.tau_c > 0.0f) {
                const float d0 = fsub(sc[i][0], m0), d1 = fsub(sc[i][1], m1), d2 = fsub(sc[i][2], m2);
                if (!(dot3(d0, d1, d2, d0, d1, d2) <= tau2)) continue;
            }
            acc0 = ffma(sw[i], sc[i][0], acc0);
            acc1 = ffma(sw[i], sc[i][1], acc1);
            acc2 = ffma(sw[i], sc[i][2], acc2);
            ws = fadd(ws, sw[i]);
        }
    }
    // Eq. 10; no weight at all is a hole even when w_min = 0 (holes are colour 0)
    float o0 = 0.0f, o1 = 0.0f, o2 = 0.0f;
    if (ws > 0.0f && ws >= bt.w_min) {
        o0 = fdiv(acc0, ws); o1 = fdiv(acc1, ws); o2 = fdiv(acc2, ws);
    }
    rgb[(size_t)pix * 3 + 0] = o0;
    rgb[(size_t)pix * 3 + 1] = o1;
    rgb[(size_t)pix * 3 + 2] = o2;
    if (wsum) wsum[pix] = ws;
}

}  // namespace ta
