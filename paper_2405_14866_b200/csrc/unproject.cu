// unproject.cu -- a1: lift foreground source pixels to latent Gaussians (sm_100a).
//
// PAPER.md l.358 (disparity -> depth), l.374 (x, f, s, alpha; rotation = identity), l.376
// (unprojection through Pi), l.385 (foreground pixels -> pixel-aligned Gaussians).
// Two passes over the source maps: k_unproject_count counts valid pixels per 1024-pixel block,
// a look-back scan turns the counts into output offsets (stable compaction: view-major,
// row-major ids), k_unproject_write recomputes validity and writes the Gaussians.  Each thread
// owns 4 consecutive pixels: disparity / opacity / scale / quaternion / feature rows are read
// with 128-bit loads when the view allows it (H*W % 4 == 0 and 16-byte aligned maps).
#include "common.cuh"
#include "internal.h"
#include "project.cuh"

namespace ta {

__device__ __forceinline__ int find_view(const ViewTable& vt, uint32_t blk) {
    int v = 0;
#pragma unroll 1
    for (int k = 1; k < vt.V; k++)
        if (blk >= vt.v[k].blk_begin) v = k;
    return v;
}

struct PixelIn {
    float d, a;
    bool m;
};

__device__ __forceinline__ void load4(const ViewDesc& vd, int64_t p0, int64_t HW, const ViewTable& vt, PixelIn in[4]) {
    if (vd.vec4 && p0 + 3 < HW) {
        const float4 d = __ldg(reinterpret_cast<const float4*>(vd.disp + p0));
        in[0].d = d.x; in[1].d = d.y; in[2].d = d.z; in[3].d = d.w;
        if (vd.opacity) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(vd.opacity + p0));
            in[0].a = a.x; in[1].a = a.y; in[2].a = a.z; in[3].a = a.w;
        } else {
            for (int k = 0; k < 4; k++) in[k].a = vt.default_opacity;
        }
        if (vd.mask) {
            const uchar4 m = __ldg(reinterpret_cast<const uchar4*>(vd.mask + p0));
            in[0].m = m.x != 0; in[1].m = m.y != 0; in[2].m = m.z != 0; in[3].m = m.w != 0;
        } else {
            for (int k = 0; k < 4; k++) in[k].m = true;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int64_t p = p0 + k;
            if (p < HW) {
                in[k].d = __ldg(vd.disp + p);
                in[k].a = vd.opacity ? __ldg(vd.opacity + p) : vt.default_opacity;
                in[k].m = vd.mask ? (__ldg(vd.mask + p) != 0) : true;
            } else {
                in[k].d = 0.0f; in[k].a = 0.0f; in[k].m = false;
            }
        }
    }
}

__device__ __forceinline__ bool pixel_valid(const PixelIn& in, float d_min) {
    return in.m && isfinite(in.d) && in.d > d_min && !isnan(in.a);
}

// a1 for one valid pixel p of view vd (normative sequence of DESIGN.md a1): world position + opacity,
// world covariance Sigma_w = R_q diag(s^2) R_q^T (upper triangle), and the id in c1.z.
__device__ __forceinline__ void lift_one(const ViewDesc& vd, const ViewTable& vt, int64_t p, const PixelIn& in, uint32_t id,
                                         float4& pa, float4& c0, float4& c1) {
    const float* R = vd.R;
    const int y = (int)(p / vd.W), x = (int)(p - (int64_t)y * vd.W);
    const float d = in.d;
    const float a = fminf(fmaxf(in.a, 0.0f), 1.0f);
    // depth (R2) and camera-space point, then X_w = R^T (X_c - t)
    const float z = fdiv(fmul(vd.fx, vd.baseline), d);
    const float xc = fmul(fdiv(fsub((float)x, vd.cx), vd.fx), z);
    const float yc = fmul(fdiv(fsub((float)y, vd.cy), vd.fy), z);
    const float q0 = fsub(xc, vd.t[0]), q1 = fsub(yc, vd.t[1]), q2 = fsub(z, vd.t[2]);
    const float w0 = dot3(R[0], R[3], R[6], q0, q1, q2);
    const float w1 = dot3(R[1], R[4], R[7], q0, q1, q2);
    const float w2 = dot3(R[2], R[5], R[8], q0, q1, q2);
    float s0, s1, s2;
    if (vd.scale) {
        s0 = __ldg(vd.scale + 3 * p + 0); s1 = __ldg(vd.scale + 3 * p + 1); s2 = __ldg(vd.scale + 3 * p + 2);
    } else {
        s0 = s1 = s2 = vt.default_scale;
    }
    float qw = 1.0f, qx = 0.0f, qy = 0.0f, qz = 0.0f;
    if (vd.quat) {
        const float4 qq = vd.vec4 ? __ldg(reinterpret_cast<const float4*>(vd.quat + 4 * p))
                                  : make_float4(__ldg(vd.quat + 4 * p), __ldg(vd.quat + 4 * p + 1),
                                                __ldg(vd.quat + 4 * p + 2), __ldg(vd.quat + 4 * p + 3));
        const float n2 = ffma(qq.w, qq.w, ffma(qq.z, qq.z, ffma(qq.y, qq.y, fmul(qq.x, qq.x))));
        if (n2 > 0.0f && isfinite(n2)) {
            const float nn = fsqrt(n2);
            qw = fdiv(qq.x, nn); qx = fdiv(qq.y, nn); qy = fdiv(qq.z, nn); qz = fdiv(qq.w, nn);
        }
    }
    const float xx = fmul(qx, qx), yy = fmul(qy, qy), zz = fmul(qz, qz);
    const float xy = fmul(qx, qy), xz = fmul(qx, qz), yz = fmul(qy, qz);
    const float wx = fmul(qw, qx), wy = fmul(qw, qy), wz = fmul(qw, qz);
    float Rq[9];
    Rq[0] = fsub(1.0f, fmul(2.0f, fadd(yy, zz))); Rq[1] = fmul(2.0f, fsub(xy, wz)); Rq[2] = fmul(2.0f, fadd(xz, wy));
    Rq[3] = fmul(2.0f, fadd(xy, wz)); Rq[4] = fsub(1.0f, fmul(2.0f, fadd(xx, zz))); Rq[5] = fmul(2.0f, fsub(yz, wx));
    Rq[6] = fmul(2.0f, fsub(xz, wy)); Rq[7] = fmul(2.0f, fadd(yz, wx)); Rq[8] = fsub(1.0f, fmul(2.0f, fadd(xx, yy)));
    const float ss[3] = {fmul(s0, s0), fmul(s1, s1), fmul(s2, s2)};
    float M[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int kk = 0; kk < 3; kk++) M[i * 3 + kk] = fmul(Rq[i * 3 + kk], ss[kk]);
    const float c00 = dot3(M[0], M[1], M[2], Rq[0], Rq[1], Rq[2]);
    const float c01 = dot3(M[0], M[1], M[2], Rq[3], Rq[4], Rq[5]);
    const float c02 = dot3(M[0], M[1], M[2], Rq[6], Rq[7], Rq[8]);
    const float c11 = dot3(M[3], M[4], M[5], Rq[3], Rq[4], Rq[5]);
    const float c12 = dot3(M[3], M[4], M[5], Rq[6], Rq[7], Rq[8]);
    const float c22 = dot3(M[6], M[7], M[8], Rq[6], Rq[7], Rq[8]);
    pa = make_float4(w0, w1, w2, a);
    c0 = make_float4(c00, c01, c02, c11);
    c1 = make_float4(c12, c22, __uint_as_float(id), 0.0f);
}

// feature row copy of pixel p to Gaussian slot `out` (16-byte chunks; rows are multiples of 16 bytes)
__device__ __forceinline__ void copy_row(const ViewDesc& vd, int64_t p, int rowbytes, void* __restrict__ feat_out,
                                         uint32_t out) {
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const char*>(vd.feat) + p * rowbytes);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<char*>(feat_out) + (size_t)out * rowbytes);
    for (int b = 0; b < rowbytes / 16; b++) dst[b] = __ldg(src + b);
}

__global__ void __launch_bounds__(kUnprojThreads) k_unproject_count(ViewTable vt, uint32_t* __restrict__ counts) {
    __shared__ uint32_t s_w[kUnprojThreads / 32];
    const uint32_t blk = blockIdx.x;
    const int v = find_view(vt, blk);
    const ViewDesc& vd = vt.v[v];
    const int64_t HW = (int64_t)vd.H * vd.W;
    const int64_t p0 = (int64_t)(blk - vd.blk_begin) * kUnprojPix + 4 * threadIdx.x;
    PixelIn in[4];
    load4(vd, p0, HW, vt, in);
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) c += pixel_valid(in[k], vt.d_min) ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane_id() == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int k = 0; k < kUnprojThreads / 32; k++) s += s_w[k];
        counts[blk] = s;
    }
}

__global__ void __launch_bounds__(kUnprojThreads) k_unproject_write(ViewTable vt, const uint32_t* __restrict__ offs,
                                                                    float4* __restrict__ pos_alpha,
                                                                    float4* __restrict__ cov, void* __restrict__ feat_out) {
    __shared__ uint32_t s_w[kUnprojThreads / 32];
    const uint32_t blk = blockIdx.x;
    const int v = find_view(vt, blk);
    const ViewDesc& vd = vt.v[v];
    const int64_t HW = (int64_t)vd.H * vd.W;
    const int64_t p0 = (int64_t)(blk - vd.blk_begin) * kUnprojPix + 4 * threadIdx.x;
    PixelIn in[4];
    load4(vd, p0, HW, vt, in);
    bool ok[4];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) { ok[k] = pixel_valid(in[k], vt.d_min); c += ok[k] ? 1u : 0u; }
    // block exclusive scan of per-thread counts
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
    for (uint32_t k = 0; k < warp; k++) wbase += s_w[k];
    uint32_t out = offs[blk] + wbase + incl - c;
    if (c == 0) return;

    const int C = vt.C;
    const int rowbytes = C * vt.fbytes;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (!ok[k]) continue;
        float4 pa, c0, c1;
        lift_one(vd, vt, p0 + k, in[k], out, pa, c0, c1);
        pos_alpha[out] = pa;
        cov[2 * (size_t)out] = c0;
        cov[2 * (size_t)out + 1] = c1;
        copy_row(vd, p0 + k, rowbytes, feat_out, out);
        out++;
    }
}

// north_star (a): fused unproject + project + cull straight from the source maps.  Same block layout
// and compaction as k_unproject_write (k_unproject_count + scan give the offsets, so Gaussian slot =
// id = the ta_unproject id), but the lifted Gaussian stays in registers: only its fp16/fp32 feature row
// is written (the compositor's operand), and it is projected into every target at once, writing each
// target's 32-byte splat record, depth key and index (exactly what k_project writes for the same
// Gaussian) plus per-target visibility statistics (OR / AND of visible depth keys, visible count) that
// k_init hands to the depth sort.  The 48-byte world position / covariance never touch HBM.
__global__ void __launch_bounds__(kUnprojThreads, 4) k_front_fused(ViewTable vt, const uint32_t* __restrict__ offs,
                                                                FrontTargets ft, RasterConsts rc,
                                                                void* __restrict__ feat_out, uint32_t* __restrict__ stats) {
    __shared__ uint32_t s_w[kUnprojThreads / 32];
    __shared__ uint32_t s_st[kMaxFrontTargets][3][kUnprojThreads / 32];
    const uint32_t blk = blockIdx.x;
    const int v = find_view(vt, blk);
    const ViewDesc& vd = vt.v[v];
    const int64_t HW = (int64_t)vd.H * vd.W;
    const int64_t p0 = (int64_t)(blk - vd.blk_begin) * kUnprojPix + 4 * threadIdx.x;
    PixelIn in[4];
    load4(vd, p0, HW, vt, in);
    bool ok[4];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) { ok[k] = pixel_valid(in[k], vt.d_min); c += ok[k] ? 1u : 0u; }
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
    for (uint32_t k = 0; k < warp; k++) wbase += s_w[k];
    uint32_t out = offs[blk] + wbase + incl - c;

    uint32_t kor[kMaxFrontTargets], kand[kMaxFrontTargets], kcnt[kMaxFrontTargets];
#pragma unroll
    for (int t = 0; t < kMaxFrontTargets; t++) { kor[t] = 0u; kand[t] = 0xffffffffu; kcnt[t] = 0u; }
    const int rowbytes = vt.C * vt.fbytes;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (!ok[k]) continue;
        float4 pa, c0, c1;
        lift_one(vd, vt, p0 + k, in[k], out, pa, c0, c1);
        copy_row(vd, p0 + k, rowbytes, feat_out, out);
#pragma unroll
        for (int t = 0; t < kMaxFrontTargets; t++) {
            if (t >= ft.T) break;
            bool vis = false;
            uint32_t key = kCulledKey;
            project_one(out, pa, c0, c1, ft.cam[t], rc, ft.rec[t], ft.key[t], ft.val[t], vis, key);
            if (vis) { kor[t] |= key; kand[t] &= key; kcnt[t]++; }
        }
        out++;
    }
#pragma unroll
    for (int t = 0; t < kMaxFrontTargets; t++) {
        if (t >= ft.T) break;
        const uint32_t o = __reduce_or_sync(0xffffffffu, kor[t]);
        const uint32_t a = __reduce_and_sync(0xffffffffu, kand[t]);
        const uint32_t n = __reduce_add_sync(0xffffffffu, kcnt[t]);
        if (lane == 0) { s_st[t][0][warp] = o; s_st[t][1][warp] = a; s_st[t][2][warp] = n; }
    }
    __syncthreads();
    if (threadIdx.x < (uint32_t)ft.T) {
        const int t = (int)threadIdx.x;
        uint32_t o = 0u, a = 0xffffffffu, n = 0u;
        for (int k = 0; k < kUnprojThreads / 32; k++) { o |= s_st[t][0][k]; a &= s_st[t][1][k]; n += s_st[t][2][k]; }
        if (n) {
            atomicOr(&stats[3 * t + 0], o);
            atomicAnd(&stats[3 * t + 1], a);
            atomicAdd(&stats[3 * t + 2], n);
        }
    }
}

__global__ void k_front_stats_init(uint32_t* stats, int T) {
    const int t = threadIdx.x;
    if (t < T) { stats[3 * t] = 0u; stats[3 * t + 1] = 0xffffffffu; stats[3 * t + 2] = 0u; }
}

}  // namespace ta
