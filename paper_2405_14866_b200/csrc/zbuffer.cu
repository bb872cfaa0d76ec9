// zbuffer.cu -- SURVEY 8(f) NEXT #2: cascade depth initialisation (sm_100a).
//
// the disparity of cam0 "is converted to a depth map and then lifted to a 3D point
// cloud.  These points are rasterized to the viewpoints of cam2 and cam3.  Z-buffers are extracted
// and converted back to disparity maps d_init"; SPEC.md l.86-94 (points_zbuffer) and DESIGN.md R23:
// nearest-pixel splat of radius r, per-pixel minimum camera-space z, ties to the lowest source index.
//   k_zb_clear    z-buffer words := ~0
//   k_zb_splat    4 source pixels per thread (128-bit disparity loads): lift (a1 sequence), project
//                 (a2 sequence), 64-bit atomicMin of (bits(Z) << 32 | source index) over the splat
//   k_zb_resolve  depth = Z of the minimum (0 where empty), disparity = fx_t * B_t / Z
// The 64-bit key makes the result independent of thread order: positive floats order like their
// bits, and the index breaks ties.
#include "common.cuh"
#include "internal.h"

namespace ta {

__global__ void k_zb_clear(unsigned long long* __restrict__ zk, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) zk[i] = ~0ull;
}

__global__ void __launch_bounds__(kUnprojThreads) k_zb_splat(ViewTable vt, TargetCam cam, float z_near, int radius,
                                                             unsigned long long* __restrict__ zk) {
    const uint32_t blk = blockIdx.x;
    int v = 0;
#pragma unroll 1
    for (int k = 1; k < vt.V; k++)
        if (blk >= vt.v[k].blk_begin) v = k;
    const ViewDesc& vd = vt.v[v];
    const int64_t HW = (int64_t)vd.H * vd.W;
    const int64_t p0 = (int64_t)(blk - vd.blk_begin) * kUnprojPix + 4 * threadIdx.x;
    float d[4];
    bool m[4];
    if (vd.vec4 && p0 + 3 < HW) {
        const float4 dd = __ldg(reinterpret_cast<const float4*>(vd.disp + p0));
        d[0] = dd.x; d[1] = dd.y; d[2] = dd.z; d[3] = dd.w;
        if (vd.mask) {
            const uchar4 mm = __ldg(reinterpret_cast<const uchar4*>(vd.mask + p0));
            m[0] = mm.x != 0; m[1] = mm.y != 0; m[2] = mm.z != 0; m[3] = mm.w != 0;
        } else {
            m[0] = m[1] = m[2] = m[3] = true;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int64_t p = p0 + k;
            d[k] = p < HW ? __ldg(vd.disp + p) : 0.0f;
            m[k] = p < HW && (vd.mask ? __ldg(vd.mask + p) != 0 : true);
        }
    }
    const float* R = vd.R;
    const float* Rt = cam.R;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (!(m[k] && isfinite(d[k]) && d[k] > vt.d_min)) continue;
        const int64_t p = p0 + k;
        const int y = (int)(p / vd.W), x = (int)(p - (int64_t)y * vd.W);
        // a1: depth (R2), camera-space point, X_w = R^T (X_c - t)
        const float z = fdiv(fmul(vd.fx, vd.baseline), d[k]);
        const float xc = fmul(fdiv(fsub((float)x, vd.cx), vd.fx), z);
        const float yc = fmul(fdiv(fsub((float)y, vd.cy), vd.fy), z);
        const float q0 = fsub(xc, vd.t[0]), q1 = fsub(yc, vd.t[1]), q2 = fsub(z, vd.t[2]);
        const float w0 = dot3(R[0], R[3], R[6], q0, q1, q2);
        const float w1 = dot3(R[1], R[4], R[7], q0, q1, q2);
        const float w2 = dot3(R[2], R[5], R[8], q0, q1, q2);
        // a2: target camera space, near cull, pixel centre; nearest pixel rounds half to even (R23)
        const float X = fadd(dot3(Rt[0], Rt[1], Rt[2], w0, w1, w2), cam.t[0]);
        const float Y = fadd(dot3(Rt[3], Rt[4], Rt[5], w0, w1, w2), cam.t[1]);
        const float Z = fadd(dot3(Rt[6], Rt[7], Rt[8], w0, w1, w2), cam.t[2]);
        if (!(Z > z_near)) continue;
        const float mx = ffma(cam.fx, fdiv(X, Z), cam.cx);
        const float my = ffma(cam.fy, fdiv(Y, Z), cam.cy);
        const float fpx = rintf(mx), fpy = rintf(my);
        const float rf = (float)radius;
        if (!(fpx >= -rf && fpx <= cam.Wm1f + rf && fpy >= -rf && fpy <= cam.Hm1f + rf)) continue;
        const int px = (int)fpx, py = (int)fpy;
        const unsigned long long key = ((unsigned long long)__float_as_uint(Z) << 32) | (uint32_t)(vd.idx0 + p);
        const int j0 = max(py - radius, 0), j1 = min(py + radius, cam.H - 1);
        const int i0 = max(px - radius, 0), i1 = min(px + radius, cam.W - 1);
        for (int j = j0; j <= j1; j++)
            for (int i = i0; i <= i1; i++) atomicMin(zk + (size_t)j * cam.W + i, key);
    }
}

__global__ void k_zb_resolve(const unsigned long long* __restrict__ zk, uint32_t n, float fx, float baseline,
                             float* __restrict__ depth, float* __restrict__ disp) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = zk[i];
        float z = 0.0f, dd = 0.0f;
        if (k != ~0ull) {
            z = __uint_as_float((uint32_t)(k >> 32));
            dd = fdiv(fmul(fx, baseline), z);
        }
        depth[i] = z;
        if (disp) disp[i] = dd;
    }
}

}  // namespace ta
