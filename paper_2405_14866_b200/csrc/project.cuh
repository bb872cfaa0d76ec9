// project.cuh -- a2 for one Gaussian, shared by k_project (raster.cu) and the fused front end
// (unproject.cu, k_front_fused): the normative fp32 sequence of DESIGN.md a2.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace ta {

// a2 for one Gaussian (normative sequence of DESIGN.md a2; mirrors nothing: the oracle is separate C
// code): writes its 32-byte splat record and its depth key / index by id; returns visibility + key.
__device__ __forceinline__ void project_one(uint32_t i, float4 pa, float4 c0, float4 c1, const TargetCam& cam,
                                            const RasterConsts& rc, uint4* __restrict__ rec,
                                            uint32_t* __restrict__ key0, uint32_t* __restrict__ val0, bool& vis,
                                            uint32_t& key) {
    const uint32_t id = __float_as_uint(c1.z);
    uint4 r0 = make_uint4(0u, 0u, 0u, 0u);
    uint4 r1 = make_uint4(0u, __float_as_uint(pa.w), kEmptyRect, kEmptyRect);
    const float* R = cam.R;
    const float X = fadd(dot3(R[0], R[1], R[2], pa.x, pa.y, pa.z), cam.t[0]);
    const float Y = fadd(dot3(R[3], R[4], R[5], pa.x, pa.y, pa.z), cam.t[1]);
    const float Z = fadd(dot3(R[6], R[7], R[8], pa.x, pa.y, pa.z), cam.t[2]);
    if (Z > rc.z_near) {
        const float u = fdiv(X, Z), v = fdiv(Y, Z);
        const float mx = ffma(cam.fx, u, cam.cx);
        const float my = ffma(cam.fy, v, cam.cy);
        const float J00 = fdiv(cam.fx, Z), J11 = fdiv(cam.fy, Z);
        const float J02 = -fmul(J00, u), J12 = -fmul(J11, v);
        float T0[3], T1[3];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            T0[j] = ffma(J02, R[6 + j], fmul(J00, R[0 + j]));
            T1[j] = ffma(J12, R[6 + j], fmul(J11, R[3 + j]));
        }
        // Sigma_w (symmetric): s00 s01 s02 s11 s12 s22
        const float S[9] = {c0.x, c0.y, c0.z, c0.y, c0.w, c1.x, c0.z, c1.x, c1.y};
        float M0[3], M1[3];
#pragma unroll
        for (int j = 0; j < 3; j++) {
            M0[j] = dot3(T0[0], T0[1], T0[2], S[0 + j], S[3 + j], S[6 + j]);
            M1[j] = dot3(T1[0], T1[1], T1[2], S[0 + j], S[3 + j], S[6 + j]);
        }
        const float a = fadd(dot3(M0[0], M0[1], M0[2], T0[0], T0[1], T0[2]), rc.dilation);
        const float b = dot3(M0[0], M0[1], M0[2], T1[0], T1[1], T1[2]);
        const float c = fadd(dot3(M1[0], M1[1], M1[2], T1[0], T1[1], T1[2]), rc.dilation);
        const float det = ffma(a, c, -fmul(b, b));
        if (det > 0.0f) {
            const float ca = fdiv(c, det);
            const float cb = fdiv(-b, det);
            const float cc = fdiv(a, det);
            const float hx = ffma(fmul(rc.cull_sigma, fsqrt(a)), 1.0009765625f, 0.0009765625f);
            const float hy = ffma(fmul(rc.cull_sigma, fsqrt(c)), 1.0009765625f, 0.0009765625f);
            const float fx0 = ceilf(fsub(mx, hx)), fx1 = floorf(fadd(mx, hx));
            const float fy0 = ceilf(fsub(my, hy)), fy1 = floorf(fadd(my, hy));
            if (fx0 <= cam.Wm1f && fx1 >= 0.0f && fy0 <= cam.Hm1f && fy1 >= 0.0f) {
                const int x0 = fx0 < 0.0f ? 0 : (int)fx0;
                const int x1 = fx1 > cam.Wm1f ? cam.W - 1 : (int)fx1;
                const int y0 = fy0 < 0.0f ? 0 : (int)fy0;
                const int y1 = fy1 > cam.Hm1f ? cam.H - 1 : (int)fy1;
                if (x0 <= x1 && y0 <= y1) {
                    vis = true;
                    key = __float_as_uint(Z);
                    r0 = make_uint4(__float_as_uint(mx), __float_as_uint(my), __float_as_uint(ca),
                                    __float_as_uint(fadd(cb, cb)));
                    r1 = make_uint4(__float_as_uint(cc), __float_as_uint(pa.w),
                                    (uint32_t)x0 | ((uint32_t)x1 << 16),
                                    (uint32_t)y0 | ((uint32_t)y1 << 16));
                }
            }
        }
    }
    rec[2 * i] = r0;
    rec[2 * i + 1] = r1;
    key0[id] = key;
    val0[id] = i;
}

}  // namespace ta
