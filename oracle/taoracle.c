/*
 * oracle/taoracle.c -- CPU ORACLE for the latent-Gaussian rasterizer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2405_14866_b200/, libtaloha.so) never links, imports or calls it, and the
 * two share no code, headers or constants generators.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited "P:<line>"):
 *   a1  lift foreground pixels to latent Gaussians {x, f, s, alpha}, R = I unless a
 *       rotation map is given ("four properties ... rotation ... identity",
 *       P:376 "3D positions x ... unprojected from depth maps", "foreground
 *       pixels ... lifted to pixel-aligned Gaussian points", P:358 disparity ->
 *       depth; z = fx*B/d is DESIGN.md reading R2);
 *   a2  project each Gaussian to the target camera Pi_novel with the EWA 2D
 *       covariance (the rasterizer of [kerbl20233d]);
 *   a3-a5  bin to 16x16 tiles and order each tile's list by (depth, id)
 *       (the [kerbl20233d] tile/sort scheme);
 *   a6  front-to-back alpha compositing of the C-channel latent feature into
 *       F_novel and accumulated alpha ("F_novel = R_G({G}, Pi_novel)").
 * Every constant the paper leaves to [kerbl20233d] is a DESIGN.md reading (R7-R13).
 *
 * Arithmetic: plain IEEE fp32, one operation at a time, in the normative order
 * written in DESIGN.md "Normative arithmetic" (built with -ffp-contract=off
 * -fno-fast-math, so every `a*b+c` below is two roundings and fmaf() is the only
 * fused operation).  Decisions that turn floats into integers (cull, pixel/tile
 * rectangles, depth order, q <= 9, alpha' >= 1/255, the T < 1e-4 stop) are taken
 * in this fp32 sequence -- the kernel's precision -- so tile lists, order and T/A
 * can be compared bit-exactly.  oracle/definition64.py is an
 * independent float64 model of the same definition that pins this file.
 *
 * Deliberately slow: qsort for the tile order, one pixel at a time for compositing.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { float fx, fy, cx, cy; } tao_intr;          /* pixels */
typedef struct { float R[9]; float t[3]; } tao_extr;        /* world->camera, R row-major */
typedef struct {
    float dilation;        /* R7: added to the diagonal of Sigma' (px^2), default 0.3 */
    float alpha_max;       /* R9: alpha' clamp, default 0.99 */
    float alpha_min;       /* R9: skip alpha' < 1/255 */
    float t_eps;           /* R10: stop before T would drop below 1e-4 */
    float cull_sigma;      /* R8: q <= cull_sigma^2 and the 3-sigma box */
    float z_near;          /* R14: cull z <= 0.01 m */
    float d_min;           /* a1: lift iff d > d_min */
    float default_scale;   /* a1: isotropic scale when no scale map */
    float default_opacity; /* a1: opacity when no opacity map */
} tao_params;

#define TAO_TILE 16

/* ------------------------------------------------------------------ helpers */

static float f16_to_f32(uint16_t h) {
    uint32_t sign = (uint32_t)(h >> 15) << 31;
    uint32_t ex = (h >> 10) & 0x1f, man = h & 0x3ff, bits;
    if (ex == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal half: renormalise */
            int e = -1;
            do { e++; man <<= 1; } while ((man & 0x400) == 0);
            bits = sign | ((uint32_t)(127 - 15 - e) << 23) | ((man & 0x3ff) << 13);
        }
    } else if (ex == 31) {
        bits = sign | 0x7f800000u | (man << 13);
    } else {
        bits = sign | ((ex + 127 - 15) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

static float feat_at(const void* feat, int feat_bytes, int C, int64_t g, int c) {
    if (feat_bytes == 2) return f16_to_f32(((const uint16_t*)feat)[g * C + c]);
    return ((const float*)feat)[g * C + c];
}

static uint32_t float_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* dot3(a, b) = fma(a2, b2, fma(a1, b1, a0*b0))  (DESIGN.md normative dot product) */
static float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return fmaf(a2, b2, fmaf(a1, b1, a0 * b0));
}

/*
 * exp_det -- DESIGN.md reading R13.  exp(x) for x <= 0 by a fixed fp32 sequence:
 * k = the integer nearest (ties to even) to the exact product x*log2 e, obtained with one
 * rounding as fma(x, log2 e, 1.5*2^23) - 1.5*2^23; reduction r = fma(-k, fl(ln 2), x) (one
 * constant: |k| <= 7 on the used range x >= -4.5, so the ln 2 rounding costs < 0.25 ulp);
 * p = 1 + r + c2 r^2 + ... + c6 r^6 (relative-error minimax on [-ln2/2, ln2/2], fp32
 * coefficients, max error 0.07 ulp) in Horner form with fmaf; scale by 2^k (exact).  Pinned in
 * tests/test_oracle_pins.py against float64 exp over [-4.5, 0] (<= 2 ulp).
 */
float tao_exp_det(float x) {
    if (x < -80.0f) x = -80.0f;
    float k = fmaf(x, 1.44269502162933349609375f, 12582912.0f) - 12582912.0f;   /* float(log2 e) */
    float r = fmaf(-k, 0.693147182464599609375f, x);                             /* float(ln 2) */
    float p = 1.3814548728987575e-3f;
    p = fmaf(p, r, 8.36869515478611e-3f);
    p = fmaf(p, r, 4.166838899254799e-2f);
    p = fmaf(p, r, 1.666652113199234e-1f);
    p = fmaf(p, r, 4.999999403953552e-1f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    uint32_t sb = (uint32_t)((int)k + 127) << 23;
    float s;
    memcpy(&s, &sb, 4);
    return p * s;
}

/* ------------------------------------------------------------ a1 unproject */
/*
 * One source view, pixels row-major.  Appends the lifted Gaussians of this view to
 * the output arrays starting at index 0 of each given pointer and returns how many.
 * ids are id0, id0+1, ... (running index over views, DESIGN.md a1).
 *   pos[n][3]  world position;   alpha[n];   cov6[n][6] = (s00,s01,s02,s11,s12,s22)
 *   ids[n];   feat_out[n][C] same element type as feat (bytes copied).
 */
int64_t tao_unproject_view(int H, int W, const float* disp, const uint8_t* mask,
                           const tao_intr* K, const tao_extr* RT, float baseline,
                           const float* scale, const float* quat, const float* opacity,
                           const void* feat, int C, int feat_bytes, const tao_params* p,
                           int64_t id0, float* pos, float* alpha, float* cov6, int64_t* ids,
                           void* feat_out) {
    int64_t n = 0;
    const float* R = RT->R;
    const float* t = RT->t;
    for (int y = 0; y < H; y++) {
        for (int x = 0; x < W; x++) {
            int64_t pix = (int64_t)y * W + x;
            float d = disp[pix];
            if (mask && mask[pix] == 0) continue;               /* foreground only */
            if (!isfinite(d) || !(d > p->d_min)) continue;      /* invalid disparity: skipped */
            float a = opacity ? opacity[pix] : p->default_opacity;
            if (isnan(a)) continue;
            a = fminf(fmaxf(a, 0.0f), 1.0f);

            /* depth from disparity (R2: z = fx*B/d) and camera-space point */
            float z = (K->fx * baseline) / d;
            float xc = (((float)x - K->cx) / K->fx) * z;
            float yc = (((float)y - K->cy) / K->fy) * z;
            float zc = z;
            /* world point X_w = R^T (X_c - t) */
            float p0 = xc - t[0], p1 = yc - t[1], p2 = zc - t[2];
            float w0 = dot3(R[0], R[3], R[6], p0, p1, p2);
            float w1 = dot3(R[1], R[4], R[7], p0, p1, p2);
            float w2 = dot3(R[2], R[5], R[8], p0, p1, p2);

            /* scale (R5) and rotation (identity; R4: optional quaternion map) */
            float s0, s1, s2;
            if (scale) { s0 = scale[pix * 3 + 0]; s1 = scale[pix * 3 + 1]; s2 = scale[pix * 3 + 2]; }
            else { s0 = s1 = s2 = p->default_scale; }
            float qw = 1.0f, qx = 0.0f, qy = 0.0f, qz = 0.0f;
            if (quat) {
                float aw = quat[pix * 4 + 0], ax = quat[pix * 4 + 1];
                float ay = quat[pix * 4 + 2], az = quat[pix * 4 + 3];
                float n2 = fmaf(az, az, fmaf(ay, ay, fmaf(ax, ax, aw * aw)));
                if (n2 > 0.0f && isfinite(n2)) {
                    float nn = sqrtf(n2);
                    qw = aw / nn; qx = ax / nn; qy = ay / nn; qz = az / nn;
                }
            }
            float xx = qx * qx, yy = qy * qy, zz = qz * qz;
            float xy = qx * qy, xz = qx * qz, yz = qy * qz;
            float wx = qw * qx, wy = qw * qy, wz = qw * qz;
            float Rq[9];
            Rq[0] = 1.0f - 2.0f * (yy + zz); Rq[1] = 2.0f * (xy - wz);        Rq[2] = 2.0f * (xz + wy);
            Rq[3] = 2.0f * (xy + wz);        Rq[4] = 1.0f - 2.0f * (xx + zz); Rq[5] = 2.0f * (yz - wx);
            Rq[6] = 2.0f * (xz - wy);        Rq[7] = 2.0f * (yz + wx);        Rq[8] = 1.0f - 2.0f * (xx + yy);
            float ss[3] = {s0 * s0, s1 * s1, s2 * s2};
            float M[9];   /* M = Rq diag(s^2) */
            for (int i = 0; i < 3; i++)
                for (int k = 0; k < 3; k++) M[i * 3 + k] = Rq[i * 3 + k] * ss[k];
            /* Sigma_w = Rq diag(s^2) Rq^T, upper triangle */
            static const int IJ[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
            for (int e = 0; e < 6; e++) {
                int i = IJ[e][0], j = IJ[e][1];
                cov6[n * 6 + e] = dot3(M[i * 3 + 0], M[i * 3 + 1], M[i * 3 + 2],
                                       Rq[j * 3 + 0], Rq[j * 3 + 1], Rq[j * 3 + 2]);
            }
            pos[n * 3 + 0] = w0; pos[n * 3 + 1] = w1; pos[n * 3 + 2] = w2;
            alpha[n] = a;
            ids[n] = id0 + n;
            memcpy((char*)feat_out + n * (int64_t)C * feat_bytes,
                   (const char*)feat + pix * (int64_t)C * feat_bytes, (size_t)C * feat_bytes);
            n++;
        }
    }
    return n;
}

/* -------------------------------------------------------------- a2 project */
/*
 * EWA projection of n Gaussians into the target camera (H x W pixels).
 * Outputs per Gaussian: visible (0/1); mean2[2] pixel centre; conic[3] =
 * (ca, cb2, cc) with q = ca dx^2 + cb2 dx dy + cc dy^2; cov2d[3] = (a, b, c) of
 * Sigma' + dilation*I; rect[4] = pixel box (x0, x1, y0, y1) inclusive; depth key
 * dkey = bits(z) of the camera-space centre depth (R12).
 */
void tao_project(int64_t n, const float* pos, const float* cov6, const tao_intr* K,
                 const tao_extr* RT, int H, int W, const tao_params* p, int32_t* visible,
                 float* mean2, float* conic, float* cov2d, int32_t* rect, uint32_t* dkey) {
    const float* R = RT->R;
    const float* t = RT->t;
    for (int64_t g = 0; g < n; g++) {
        visible[g] = 0;
        dkey[g] = 0;
        rect[g * 4 + 0] = 1; rect[g * 4 + 1] = 0; rect[g * 4 + 2] = 1; rect[g * 4 + 3] = 0;
        float w0 = pos[g * 3 + 0], w1 = pos[g * 3 + 1], w2 = pos[g * 3 + 2];
        float X = dot3(R[0], R[1], R[2], w0, w1, w2) + t[0];
        float Y = dot3(R[3], R[4], R[5], w0, w1, w2) + t[1];
        float Z = dot3(R[6], R[7], R[8], w0, w1, w2) + t[2];
        if (!(Z > p->z_near)) continue;                                   /* R14 */
        float u = X / Z, v = Y / Z;
        float mx = fmaf(K->fx, u, K->cx);
        float my = fmaf(K->fy, v, K->cy);
        /* EWA: J = d(pixel)/d(X_c) at X (2x3, J01 = J10 = 0); T = J R */
        float J00 = K->fx / Z, J11 = K->fy / Z;
        float J02 = -(J00 * u), J12 = -(J11 * v);
        float T0[3], T1[3];
        for (int j = 0; j < 3; j++) {
            T0[j] = fmaf(J02, R[6 + j], J00 * R[0 + j]);
            T1[j] = fmaf(J12, R[6 + j], J11 * R[3 + j]);
        }
        const float* s = cov6 + g * 6;
        float S[9] = {s[0], s[1], s[2], s[1], s[3], s[4], s[2], s[4], s[5]};
        float M0[3], M1[3];   /* M = T Sigma_w */
        for (int j = 0; j < 3; j++) {
            M0[j] = dot3(T0[0], T0[1], T0[2], S[0 + j], S[3 + j], S[6 + j]);
            M1[j] = dot3(T1[0], T1[1], T1[2], S[0 + j], S[3 + j], S[6 + j]);
        }
        /* Sigma' = M T^T (+ dilation on the diagonal, R7) */
        float a = dot3(M0[0], M0[1], M0[2], T0[0], T0[1], T0[2]) + p->dilation;
        float b = dot3(M0[0], M0[1], M0[2], T1[0], T1[1], T1[2]);
        float c = dot3(M1[0], M1[1], M1[2], T1[0], T1[1], T1[2]) + p->dilation;
        float det = fmaf(a, c, -(b * b));
        if (!(det > 0.0f)) continue;
        float ca = c / det;
        float cb = (-b) / det;
        float cc = a / det;
        /* 3-sigma box with rounding margin (R8), clipped to the image (R18) */
        float hx = fmaf(p->cull_sigma * sqrtf(a), 1.0009765625f, 0.0009765625f);
        float hy = fmaf(p->cull_sigma * sqrtf(c), 1.0009765625f, 0.0009765625f);
        float fx0 = ceilf(mx - hx), fx1 = floorf(mx + hx);
        float fy0 = ceilf(my - hy), fy1 = floorf(my + hy);
        if (!(fx0 <= (float)(W - 1)) || !(fx1 >= 0.0f) || !(fy0 <= (float)(H - 1)) || !(fy1 >= 0.0f))
            continue;
        int x0 = fx0 < 0.0f ? 0 : (int)fx0;
        int x1 = fx1 > (float)(W - 1) ? W - 1 : (int)fx1;
        int y0 = fy0 < 0.0f ? 0 : (int)fy0;
        int y1 = fy1 > (float)(H - 1) ? H - 1 : (int)fy1;
        if (x0 > x1 || y0 > y1) continue;
        visible[g] = 1;
        mean2[g * 2 + 0] = mx; mean2[g * 2 + 1] = my;
        conic[g * 3 + 0] = ca; conic[g * 3 + 1] = cb + cb; conic[g * 3 + 2] = cc;
        cov2d[g * 3 + 0] = a; cov2d[g * 3 + 1] = b; cov2d[g * 3 + 2] = c;
        rect[g * 4 + 0] = x0; rect[g * 4 + 1] = x1; rect[g * 4 + 2] = y0; rect[g * 4 + 3] = y1;
        dkey[g] = float_bits(Z);
    }
}

/* ----------------------------------------------------- a3-a5 tile lists */

typedef struct { uint32_t tile, dkey; int64_t id, g; } tao_entry;

static int entry_cmp(const void* pa, const void* pb) {
    const tao_entry* a = (const tao_entry*)pa;
    const tao_entry* b = (const tao_entry*)pb;
    if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
    if (a->dkey != b->dkey) return a->dkey < b->dkey ? -1 : 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return 0;
}

/* K = number of (tile, Gaussian) pairs for square screen tiles of side `tile` pixels: each visible
 * Gaussian covers the tiles of its pixel box.  The paper takes the tiling from [kerbl20233d] (PAPER.md
 * l.387: 16 x 16); the side is a free parameter of the binning -- a pixel's composited sequence (the
 * Gaussians whose box holds it, in (dkey, id) order) is the same for every side (R8). */
int64_t tao_count_entries_tiled(int64_t n, const int32_t* visible, const int32_t* rect, int tile) {
    int64_t K = 0;
    for (int64_t g = 0; g < n; g++) {
        if (!visible[g]) continue;
        int64_t tw = rect[g * 4 + 1] / tile - rect[g * 4 + 0] / tile + 1;
        int64_t th = rect[g * 4 + 3] / tile - rect[g * 4 + 2] / tile + 1;
        K += tw * th;
    }
    return K;
}

int64_t tao_count_entries(int64_t n, const int32_t* visible, const int32_t* rect) {
    return tao_count_entries_tiled(n, visible, rect, TAO_TILE);
}

/*
 * Per-tile lists ordered by (tile, dkey, id): ranges[T][2] = [start, end) into list;
 * list[K] = array index g of the Gaussian.  Tiles of side `tile` are row-major,
 * T = ceil(W/tile)*ceil(H/tile).  Returns K.
 */
int64_t tao_tile_lists_tiled(int64_t n, const int32_t* visible, const int32_t* rect, const uint32_t* dkey,
                             const int64_t* ids, int H, int W, int tile, uint32_t* ranges, int64_t* list) {
    int TX = (W + tile - 1) / tile, TY = (H + tile - 1) / tile;
    int64_t K = tao_count_entries_tiled(n, visible, rect, tile);
    tao_entry* e = (tao_entry*)malloc(sizeof(tao_entry) * (size_t)(K > 0 ? K : 1));
    int64_t k = 0;
    for (int64_t g = 0; g < n; g++) {
        if (!visible[g]) continue;
        for (int ty = rect[g * 4 + 2] / tile; ty <= rect[g * 4 + 3] / tile; ty++)
            for (int tx = rect[g * 4 + 0] / tile; tx <= rect[g * 4 + 1] / tile; tx++) {
                e[k].tile = (uint32_t)(ty * TX + tx);
                e[k].dkey = dkey[g];
                e[k].id = ids[g];
                e[k].g = g;
                k++;
            }
    }
    qsort(e, (size_t)K, sizeof(tao_entry), entry_cmp);
    for (int t = 0; t < TX * TY; t++) { ranges[2 * t] = 0; ranges[2 * t + 1] = 0; }
    for (int64_t i = 0; i < K; i++) {
        uint32_t t = e[i].tile;
        if (i == 0 || e[i - 1].tile != t) ranges[2 * t] = (uint32_t)i;
        ranges[2 * t + 1] = (uint32_t)(i + 1);
        list[i] = e[i].g;
    }
    free(e);
    return K;
}

int64_t tao_tile_lists(int64_t n, const int32_t* visible, const int32_t* rect, const uint32_t* dkey,
                       const int64_t* ids, int H, int W, uint32_t* ranges, int64_t* list) {
    return tao_tile_lists_tiled(n, visible, rect, dkey, ids, H, W, TAO_TILE, ranges, list);
}

/* ------------------------------------------------------------ a6 composite */

/* Front-to-back compositing of one pixel over a sequence of Gaussians (DESIGN.md a6). */
static void composite_pixel(int px, int py, int C, int64_t count, const int64_t* seq,
                            const float* alpha, const float* mean2, const float* conic,
                            const int32_t* rect, const void* feat, int feat_bytes,
                            const tao_params* p, float* F, float* A, int32_t* n_contrib,
                            int32_t* n_eval) {
    float T = 1.0f;
    float qmax = p->cull_sigma * p->cull_sigma;
    int32_t nc = 0, ne = 0;
    for (int c = 0; c < C; c++) F[c] = 0.0f;
    for (int64_t j = 0; j < count; j++) {
        int64_t g = seq[j];
        ne++;
        const int32_t* r = rect + g * 4;
        if (px < r[0] || px > r[1] || py < r[2] || py > r[3]) continue;   /* R8 box */
        float dx = (float)px - mean2[g * 2 + 0];
        float dy = (float)py - mean2[g * 2 + 1];
        float q = fmaf(fmaf(conic[g * 3 + 0], dx, conic[g * 3 + 1] * dy), dx,
                       (conic[g * 3 + 2] * dy) * dy);
        if (!(q <= qmax)) continue;                                         /* 3 sigma */
        float e = tao_exp_det(-0.5f * q);
        float a = fminf(p->alpha_max, alpha[g] * e);                        /* R9 */
        if (a < p->alpha_min) continue;
        float Tn = T * (1.0f - a);
        if (Tn < p->t_eps) break;                                           /* R10 */
        float w = a * T;
        for (int c = 0; c < C; c++) F[c] = F[c] + feat_at(feat, feat_bytes, C, g, c) * w;
        T = Tn;
        nc++;
    }
    *A = 1.0f - T;                                                          /* R11 */
    if (n_contrib) *n_contrib = nc;
    if (n_eval) *n_eval = ne;
}

/*
 * Tiled compositing: each pixel walks its tile's (dkey, id)-ordered list.
 * tiles: indices of the tiles to render (NULL = all).  F[H*W*C] (HWC), A[H*W];
 * n_contrib / n_eval [H*W] optional.  Pixels of tiles not rendered are untouched.
 */
void tao_composite_tiles(int H, int W, int C, int feat_bytes, const float* alpha,
                         const float* mean2, const float* conic, const int32_t* rect,
                         const void* feat, const uint32_t* ranges, const int64_t* list,
                         const tao_params* p, const int32_t* tiles, int64_t n_tiles, float* F,
                         float* A, int32_t* n_contrib, int32_t* n_eval) {
    int TX = (W + TAO_TILE - 1) / TAO_TILE, TY = (H + TAO_TILE - 1) / TAO_TILE;
    if (!tiles) n_tiles = (int64_t)TX * TY;
    for (int64_t k = 0; k < n_tiles; k++) {
        int t = tiles ? tiles[k] : (int)k;
        int tx = t % TX, ty = t / TX;
        uint32_t s = ranges[2 * t], e = ranges[2 * t + 1];
        for (int py = ty * TAO_TILE; py < ty * TAO_TILE + TAO_TILE && py < H; py++)
            for (int px = tx * TAO_TILE; px < tx * TAO_TILE + TAO_TILE && px < W; px++) {
                int64_t pix = (int64_t)py * W + px;
                composite_pixel(px, py, C, (int64_t)(e - s), list + s, alpha, mean2, conic, rect,
                                feat, feat_bytes, p, F + pix * C, A + pix,
                                n_contrib ? n_contrib + pix : NULL, n_eval ? n_eval + pix : NULL);
            }
    }
}

typedef struct { uint32_t dkey; int64_t id, g; } tao_depth;

static int depth_cmp(const void* pa, const void* pb) {
    const tao_depth* a = (const tao_depth*)pa;
    const tao_depth* b = (const tao_depth*)pb;
    if (a->dkey != b->dkey) return a->dkey < b->dkey ? -1 : 1;
    if (a->id != b->id) return a->id < b->id ? -1 : 1;
    return 0;
}

/*
 * Brute force: no tiles.  Every pixel walks ALL visible Gaussians in global (dkey, id)
 * order with the same inclusion predicate.  rows [y0, y1) only (row bands bound time).
 */
void tao_composite_bruteforce(int H, int W, int C, int feat_bytes, int64_t n,
                              const int32_t* visible, const uint32_t* dkey, const int64_t* ids,
                              const float* alpha, const float* mean2, const float* conic,
                              const int32_t* rect, const void* feat, const tao_params* p,
                              int y0, int y1, float* F, float* A, int32_t* n_contrib) {
    int64_t m = 0;
    tao_depth* d = (tao_depth*)malloc(sizeof(tao_depth) * (size_t)(n > 0 ? n : 1));
    for (int64_t g = 0; g < n; g++)
        if (visible[g]) { d[m].dkey = dkey[g]; d[m].id = ids[g]; d[m].g = g; m++; }
    qsort(d, (size_t)m, sizeof(tao_depth), depth_cmp);
    int64_t* seq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t i = 0; i < m; i++) seq[i] = d[i].g;
    free(d);
    for (int py = y0; py < y1 && py < H; py++)
        for (int px = 0; px < W; px++) {
            int64_t pix = (int64_t)py * W + px;
            composite_pixel(px, py, C, m, seq, alpha, mean2, conic, rect, feat, feat_bytes, p,
                            F + pix * C, A + pix, n_contrib ? n_contrib + pix : NULL, NULL);
        }
    free(seq);
}

/* vectorised exp_det for the pins */
void tao_exp_det_array(int64_t n, const float* x, float* y) {
    for (int64_t i = 0; i < n; i++) y[i] = tao_exp_det(x[i]);
}

/* ----------------------------------------------- NEXT: cascade Z-buffer */
/*
 * "The predicted disparity of cam0 is converted to a depth map and then
 * lifted to a 3D point cloud.  These points are rasterized to the viewpoints of cam2 and cam3.
 * Z-buffers are extracted and converted back to disparity maps d_init."
 * (points_zbuffer): per-pixel minimum camera-space z of all points splatted nearest-pixel with a
 * splat radius r (default 1 px); pixels with no point are invalid; min-z with tie-break by the
 * lowest source-pixel index.  DESIGN.md reading R23 fixes the arithmetic: lifting
 * is the a1 sequence (z = fx*B/d, X_w = R^T (X_c - t)), projection the a2 sequence
 * (X = R X_w + t, cull Z <= z_near, mu = fma(f, X/Z, c)), nearest pixel = rintf(mu) (ties to even),
 * splat to every pixel of [px - r, px + r] x [py - r, py + r] inside the target.
 *
 * One source view: lifts its valid pixels (mask != 0, finite d > d_min) and min-accumulates the
 * 64-bit key (bits(Z) << 32 | source index) into zkey[Ht*Wt] (caller fills it with ~0 first).
 * Source index = idx0 + y*W + x (idx0: running pixel offset over the views).
 */
void tao_zbuffer_view(int H, int W, const float* disp, const uint8_t* mask, const tao_intr* K,
                      const tao_extr* RT, float baseline, const tao_params* p, int64_t idx0,
                      const tao_intr* Kt, const tao_extr* RTt, int Ht, int Wt, int r, uint64_t* zkey) {
    const float* R = RT->R;
    const float* t = RT->t;
    const float* Rt = RTt->R;
    const float* tt = RTt->t;
    for (int y = 0; y < H; y++) {
        for (int x = 0; x < W; x++) {
            int64_t pix = (int64_t)y * W + x;
            float d = disp[pix];
            if (mask && mask[pix] == 0) continue;
            if (!isfinite(d) || !(d > p->d_min)) continue;
            /* a1: depth, camera-space point, world point */
            float z = (K->fx * baseline) / d;
            float xc = (((float)x - K->cx) / K->fx) * z;
            float yc = (((float)y - K->cy) / K->fy) * z;
            float p0 = xc - t[0], p1 = yc - t[1], p2 = z - t[2];
            float w0 = dot3(R[0], R[3], R[6], p0, p1, p2);
            float w1 = dot3(R[1], R[4], R[7], p0, p1, p2);
            float w2 = dot3(R[2], R[5], R[8], p0, p1, p2);
            /* a2: target camera space, cull, pixel centre */
            float X = dot3(Rt[0], Rt[1], Rt[2], w0, w1, w2) + tt[0];
            float Y = dot3(Rt[3], Rt[4], Rt[5], w0, w1, w2) + tt[1];
            float Z = dot3(Rt[6], Rt[7], Rt[8], w0, w1, w2) + tt[2];
            if (!(Z > p->z_near)) continue;
            float mx = fmaf(Kt->fx, X / Z, Kt->cx);
            float my = fmaf(Kt->fy, Y / Z, Kt->cy);
            float fpx = rintf(mx), fpy = rintf(my);
            if (!(fpx >= (float)(-r) && fpx <= (float)(Wt - 1 + r) && fpy >= (float)(-r) && fpy <= (float)(Ht - 1 + r)))
                continue;
            int px = (int)fpx, py = (int)fpy;
            uint64_t key = ((uint64_t)float_bits(Z) << 32) | (uint64_t)(uint32_t)(idx0 + pix);
            for (int j = py - r; j <= py + r; j++) {
                if (j < 0 || j >= Ht) continue;
                for (int i = px - r; i <= px + r; i++) {
                    if (i < 0 || i >= Wt) continue;
                    uint64_t* zk = zkey + (int64_t)j * Wt + i;
                    if (key < *zk) *zk = key;
                }
            }
        }
    }
}

/* Z-buffer -> depth (Z of the nearest point, 0 where none) and disparity fx*B/Z (0 where none). */
void tao_zbuffer_resolve(int64_t n, const uint64_t* zkey, float fx, float baseline, float* depth, float* dispo) {
    for (int64_t i = 0; i < n; i++) {
        if (zkey[i] == ~(uint64_t)0) { depth[i] = 0.0f; if (dispo) dispo[i] = 0.0f; continue; }
        uint32_t zb = (uint32_t)(zkey[i] >> 32);
        float z;
        memcpy(&z, &zb, 4);
        depth[i] = z;
        if (dispo) dispo[i] = (fx * baseline) / z;
    }
}

/* ------------------------------------- NEXT: occlusion-aware input-view blending */
/*
 * PAPER.md l.420-444 (Eqs. 6-10): each pixel of the fused depth z_fused (the min-z warp of all
 * input depth maps into the novel view, tao_zbuffer_view) is lifted (Pi_novel^-1) and projected into
 * every input view i (Eq. 6); colour c_i and depth z_i are bilinearly sampled there (Eq. 7); the
 * weight is w_i = M_i(x_i.uv) * Occ(x_i) * cos<r(u,v), n_i> / ||x_i^cam|| (Eq. 8) with
 * Occ = [|x_i.z - z_i| < delta] (Eq. 9); I_blend = sum w_i c_i / sum w_i (Eq. 10).
 * reading R24 fixes what the paper leaves open, in this order:
 *   - input depth z = fx*B/d where the pixel is valid (mask != 0, finite d > d_min), as in a1;
 *   - sample valid iff the projected centre lies inside [0, W-1] x [0, H-1] and Z > z_near;
 *     bilinear taps x0 = min(floor(u), W-2) (0 when W == 1), x1 = min(x0+1, W-1), likewise y;
 *     lerp(a, b, t) = fma(t, b - a, a), rows first; all four depth taps must be valid;
 *   - M_i: the input mask (through tap validity), the edge mask max(|z_r - z_l|, |z_d - z_u|)/2
 *     <= edge_tau at the nearest pixel rint(x_i.uv), a valid normal there (4 neighbours valid), and the
 *     appearance-consistency mask of l.433 (not defined by the paper; SPEC.md l.331's reading): over
 *     the samples that pass everything else (weight w_i > 0), m = the weighted median sample (the
 *     weighted medoid: the c_i minimising sum_j w_j |c_j - c_i|_2, ties to the lower view index), and a
 *     sample is kept iff |c_i - m|^2 <= tau_c^2 (tau_c = 0: mask off) -- a first pass computes every
 *     w_i, c_i and m, a second one blends; the medoid itself is always kept;
 *   - n_i: cross product of the central differences of the lifted camera-space points
 *     (SPEC.md l.120), normalised, flipped to face camera i, rotated to world (R_i^T n);
 *   - cos<r, n_i> = max(0, -r_hat . n_w) with r_hat the unit ray from the novel centre to the point;
 *   - ||x_i^cam|| = the Euclidean norm of the point in camera i's frame;
 *   - views accumulate in index order; sum w < w_min -> hole: colour 0.
 * Outputs: rgb[H][W][3], wsum[H][W] (the denominator, 0 on holes of z_fused).
 */
typedef struct {
    int H, W;
    const float* disp;
    const uint8_t* mask;
    tao_intr K;
    tao_extr RT;
    float baseline;
    const float* color;   /* [H][W][3] */
} tao_bview;

typedef struct { float delta, edge_tau, w_min, tau_c; } tao_bparams;
#define TAO_MAX_BLEND_VIEWS 16

static int bview_depth(const tao_bview* v, int x, int y, const tao_params* p, float* z) {
    if (x < 0 || y < 0 || x >= v->W || y >= v->H) return 0;
    int64_t i = (int64_t)y * v->W + x;
    if (v->mask && v->mask[i] == 0) return 0;
    float d = v->disp[i];
    if (!isfinite(d) || !(d > p->d_min)) return 0;
    *z = (v->K.fx * v->baseline) / d;
    return 1;
}

static float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

void tao_blend(int V, const tao_bview* views, const tao_params* p, const tao_bparams* bp, const tao_intr* K,
               const tao_extr* RT, int H, int W, const float* zf, float* rgb, float* wsum) {
    if (V > TAO_MAX_BLEND_VIEWS) V = TAO_MAX_BLEND_VIEWS;
    const float* R = RT->R;
    const float* t = RT->t;
    /* novel camera centre C = R^T (0 - t) */
    float c0 = dot3(R[0], R[3], R[6], -t[0], -t[1], -t[2]);
    float c1 = dot3(R[1], R[4], R[7], -t[0], -t[1], -t[2]);
    float c2 = dot3(R[2], R[5], R[8], -t[0], -t[1], -t[2]);
    for (int v = 0; v < H; v++) {
        for (int u = 0; u < W; u++) {
            int64_t pix = (int64_t)v * W + u;
            float acc[3] = {0.0f, 0.0f, 0.0f}, ws = 0.0f;
            float sw[TAO_MAX_BLEND_VIEWS], sc[TAO_MAX_BLEND_VIEWS][3];   /* pass 1: every view's w_i, c_i */
            int ns = 0;
            float z = zf[pix];
            if (z > 0.0f) {
                /* Eq. 6: Pi_novel^-1(u, v, z_fused) */
                float xc = (((float)u - K->cx) / K->fx) * z;
                float yc = (((float)v - K->cy) / K->fy) * z;
                float q0 = xc - t[0], q1 = yc - t[1], q2 = z - t[2];
                float w0 = dot3(R[0], R[3], R[6], q0, q1, q2);
                float w1 = dot3(R[1], R[4], R[7], q0, q1, q2);
                float w2 = dot3(R[2], R[5], R[8], q0, q1, q2);
                float r0 = w0 - c0, r1 = w1 - c1, r2 = w2 - c2;
                float rl = sqrtf(dot3(r0, r1, r2, r0, r1, r2));
                r0 = r0 / rl; r1 = r1 / rl; r2 = r2 / rl;
                for (int i = 0; i < V; i++) {
                    const tao_bview* bv = views + i;
                    const float* Ri = bv->RT.R;
                    const float* ti = bv->RT.t;
                    float X = dot3(Ri[0], Ri[1], Ri[2], w0, w1, w2) + ti[0];
                    float Y = dot3(Ri[3], Ri[4], Ri[5], w0, w1, w2) + ti[1];
                    float Z = dot3(Ri[6], Ri[7], Ri[8], w0, w1, w2) + ti[2];
                    if (!(Z > p->z_near)) continue;
                    float us = fmaf(bv->K.fx, X / Z, bv->K.cx);
                    float vs = fmaf(bv->K.fy, Y / Z, bv->K.cy);
                    if (!(us >= 0.0f && us <= (float)(bv->W - 1) && vs >= 0.0f && vs <= (float)(bv->H - 1))) continue;
                    /* Eq. 7: bilinear taps */
                    int x0 = (int)floorf(us), y0 = (int)floorf(vs);
                    if (x0 > bv->W - 2) x0 = bv->W >= 2 ? bv->W - 2 : 0;
                    if (y0 > bv->H - 2) y0 = bv->H >= 2 ? bv->H - 2 : 0;
                    int x1 = x0 + 1 < bv->W ? x0 + 1 : x0, y1 = y0 + 1 < bv->H ? y0 + 1 : y0;
                    float ax = us - (float)x0, ay = vs - (float)y0;
                    float z00, z10, z01, z11;
                    if (!bview_depth(bv, x0, y0, p, &z00) || !bview_depth(bv, x1, y0, p, &z10) ||
                        !bview_depth(bv, x0, y1, p, &z01) || !bview_depth(bv, x1, y1, p, &z11))
                        continue;
                    float zs = lerpf(lerpf(z00, z10, ax), lerpf(z01, z11, ax), ay);
                    /* Eq. 9: occlusion (SDF) check */
                    if (!(fabsf(Z - zs) < bp->delta)) continue;
                    /* M_i edge mask + normal at the nearest pixel */
                    int px = (int)rintf(us), py = (int)rintf(vs);
                    float zc, zl, zr, zu, zd;
                    if (!bview_depth(bv, px, py, p, &zc) || !bview_depth(bv, px - 1, py, p, &zl) ||
                        !bview_depth(bv, px + 1, py, p, &zr) || !bview_depth(bv, px, py - 1, p, &zu) ||
                        !bview_depth(bv, px, py + 1, p, &zd))
                        continue;
                    if (fmaxf(fabsf(zr - zl), fabsf(zd - zu)) * 0.5f > bp->edge_tau) continue;
                    const tao_intr* Ki = &bv->K;
                    float lx = (((float)(px - 1) - Ki->cx) / Ki->fx) * zl, ly = (((float)py - Ki->cy) / Ki->fy) * zl;
                    float rx = (((float)(px + 1) - Ki->cx) / Ki->fx) * zr, ry = (((float)py - Ki->cy) / Ki->fy) * zr;
                    float ux = (((float)px - Ki->cx) / Ki->fx) * zu, uy = (((float)(py - 1) - Ki->cy) / Ki->fy) * zu;
                    float dx = (((float)px - Ki->cx) / Ki->fx) * zd, dy = (((float)(py + 1) - Ki->cy) / Ki->fy) * zd;
                    float tx0 = rx - lx, tx1 = ry - ly, tx2 = zr - zl;
                    float ty0 = dx - ux, ty1 = dy - uy, ty2 = zd - zu;
                    float n0 = fmaf(tx1, ty2, -(tx2 * ty1));
                    float n1 = fmaf(tx2, ty0, -(tx0 * ty2));
                    float n2 = fmaf(tx0, ty1, -(tx1 * ty0));
                    float nl = sqrtf(dot3(n0, n1, n2, n0, n1, n2));
                    if (!(nl > 0.0f)) continue;
                    n0 = n0 / nl; n1 = n1 / nl; n2 = n2 / nl;
                    float pcx = (((float)px - Ki->cx) / Ki->fx) * zc, pcy = (((float)py - Ki->cy) / Ki->fy) * zc;
                    if (dot3(n0, n1, n2, pcx, pcy, zc) > 0.0f) { n0 = -n0; n1 = -n1; n2 = -n2; }
                    float m0 = dot3(Ri[0], Ri[3], Ri[6], n0, n1, n2);
                    float m1 = dot3(Ri[1], Ri[4], Ri[7], n0, n1, n2);
                    float m2 = dot3(Ri[2], Ri[5], Ri[8], n0, n1, n2);
                    /* Eq. 8 */
                    float cs = -dot3(r0, r1, r2, m0, m1, m2);
                    if (!(cs > 0.0f)) continue;
                    float dist = sqrtf(dot3(X, Y, Z, X, Y, Z));
                    float w = cs / dist;
                    const float* col = bv->color;
                    for (int k = 0; k < 3; k++) {
                        float a00 = col[((int64_t)y0 * bv->W + x0) * 3 + k], a10 = col[((int64_t)y0 * bv->W + x1) * 3 + k];
                        float a01 = col[((int64_t)y1 * bv->W + x0) * 3 + k], a11 = col[((int64_t)y1 * bv->W + x1) * 3 + k];
                        sc[ns][k] = lerpf(lerpf(a00, a10, ax), lerpf(a01, a11, ax), ay);
                    }
                    sw[ns++] = w;
                }
                /* appearance consistency: m = the weighted median sample (medoid): the c_i
                   minimising sum_j w_j |c_j - c_i| (sums in view order, ties to the lower index) */
                float m[3] = {0.0f, 0.0f, 0.0f};
                if (bp->tau_c > 0.0f && ns > 0) {
                    float best = INFINITY;
                    int bi = 0;
                    for (int i = 0; i < ns; i++) {
                        float cost = 0.0f;
                        for (int j = 0; j < ns; j++) {
                            float e0 = sc[j][0] - sc[i][0], e1 = sc[j][1] - sc[i][1], e2 = sc[j][2] - sc[i][2];
                            cost = fmaf(sw[j], sqrtf(dot3(e0, e1, e2, e0, e1, e2)), cost);
                        }
                        if (cost < best) { best = cost; bi = i; }
                    }
                    for (int k = 0; k < 3; k++) m[k] = sc[bi][k];
                }
                const float tau2 = bp->tau_c * bp->tau_c;
                /* pass 2: Eq. 10 sums over the consistent samples, in view order */
                for (int i = 0; i < ns; i++) {
                    if (bp->tau_c > 0.0f) {
                        float d0 = sc[i][0] - m[0], d1 = sc[i][1] - m[1], d2 = sc[i][2] - m[2];
                        if (!(dot3(d0, d1, d2, d0, d1, d2) <= tau2)) continue;
                    }
                    for (int k = 0; k < 3; k++) acc[k] = fmaf(sw[i], sc[i][k], acc[k]);
                    ws = ws + sw[i];
                }
            }
            /* Eq. 10; sum w = 0 is a hole even for w_min = 0 (hole colour 0) */
            if (ws > 0.0f && ws >= bp->w_min) {
                for (int k = 0; k < 3; k++) rgb[pix * 3 + k] = acc[k] / ws;
            } else {
                for (int k = 0; k < 3; k++) rgb[pix * 3 + k] = 0.0f;
            }
            if (wsum) wsum[pix] = ws;
        }
    }
}

/* --------------------------------------------- NEXT: compositing backward pass */
/*
 * Gradients of L = sum_p G_F(p) . F(p) + G_A(p) A(p) with respect to each Gaussian's 2D splat
 * parameters (mean2, conic (ca, cb2, cc) as in the records, alpha) and its feature row, for the a6
 * forward of P:386 (the differentiable rasterizer of [kerbl20233d]).  DESIGN.md reading R25:
 * the per-pixel decisions (box, q <= q_max, alpha' >= alpha_min, the stop) are piecewise constant in
 * the parameters and held fixed; the clamp alpha' = min(alpha_max, alpha e) passes no gradient where
 * it binds.  With w_j = alpha'_j T_j, g_j = G_F . f_j, S = sum_j w_j g_j, T_end = T after the last
 * composited entry:
 *   dL/df_j      += w_j G_F
 *   dL/dalpha'_j  = T_j g_j - (S - sum_{k<=j} w_k g_k) / (1 - alpha'_j) + G_A T_end / (1 - alpha'_j)
 *   dL/dalpha_j  += dL/dalpha'_j e_j (unclamped);  dL/dq_j = dL/dalpha'_j alpha_j (-e_j / 2)
 *   dL/d(ca, cb2, cc) += dL/dq (dx^2, dx dy, dy^2);  dL/dmean2 += dL/dq (-(2 ca dx + cb2 dy), -(cb2 dx + 2 cc dy))
 * Per-pixel terms in fp32 following the forward sequence; the sums over pixels in double.
 */
void tao_composite_backward(int H, int W, int C, int feat_bytes, const float* alpha, const float* mean2,
                            const float* conic, const int32_t* rect, const void* feat, const uint32_t* ranges,
                            const int64_t* list, const tao_params* p, const float* GF, const float* GA,
                            double* d_mean2, double* d_conic, double* d_alpha, double* d_feat) {
    int TX = (W + TAO_TILE - 1) / TAO_TILE, TY = (H + TAO_TILE - 1) / TAO_TILE;
    float qmax = p->cull_sigma * p->cull_sigma;
    int64_t maxlen = 1;
    for (int t = 0; t < TX * TY; t++)
        if ((int64_t)(ranges[2 * t + 1] - ranges[2 * t]) > maxlen) maxlen = ranges[2 * t + 1] - ranges[2 * t];
    int64_t* cg = (int64_t*)malloc(sizeof(int64_t) * (size_t)maxlen);
    float* ca_ = (float*)malloc(sizeof(float) * (size_t)maxlen * 6);   /* a', T, e, dx, dy, clamped */
    for (int t = 0; t < TX * TY; t++) {
        int tx = t % TX, ty = t / TX;
        uint32_t s0 = ranges[2 * t], s1 = ranges[2 * t + 1];
        for (int py = ty * TAO_TILE; py < ty * TAO_TILE + TAO_TILE && py < H; py++)
            for (int px = tx * TAO_TILE; px < tx * TAO_TILE + TAO_TILE && px < W; px++) {
                int64_t pix = (int64_t)py * W + px;
                const float* gf = GF + pix * C;
                /* forward (the a6 sequence): the composited entries and their T, alpha', e */
                float T = 1.0f;
                int64_t m = 0;
                for (uint32_t k = s0; k < s1; k++) {
                    int64_t g = list[k];
                    const int32_t* r = rect + g * 4;
                    if (px < r[0] || px > r[1] || py < r[2] || py > r[3]) continue;
                    float dx = (float)px - mean2[g * 2 + 0];
                    float dy = (float)py - mean2[g * 2 + 1];
                    float q = fmaf(fmaf(conic[g * 3 + 0], dx, conic[g * 3 + 1] * dy), dx, (conic[g * 3 + 2] * dy) * dy);
                    if (!(q <= qmax)) continue;
                    float e = tao_exp_det(-0.5f * q);
                    float ae = alpha[g] * e;
                    float a = fminf(p->alpha_max, ae);
                    if (a < p->alpha_min) continue;
                    float Tn = T * (1.0f - a);
                    if (Tn < p->t_eps) break;
                    cg[m] = g;
                    float* rec = ca_ + m * 6;
                    rec[0] = a; rec[1] = T; rec[2] = e; rec[3] = dx; rec[4] = dy; rec[5] = ae > p->alpha_max ? 1.0f : 0.0f;
                    m++;
                    T = Tn;
                }
                float Tend = T;
                /* S = sum w_j g_j */
                float S = 0.0f;
                for (int64_t j = 0; j < m; j++) {
                    int64_t g = cg[j];
                    float gj = 0.0f;
                    for (int c = 0; c < C; c++) gj = fmaf(gf[c], feat_at(feat, feat_bytes, C, g, c), gj);
                    S = fmaf(ca_[j * 6 + 0] * ca_[j * 6 + 1], gj, S);
                }
                float Sup = 0.0f, ga = GA[pix];
                for (int64_t j = 0; j < m; j++) {
                    int64_t g = cg[j];
                    const float* rec = ca_ + j * 6;
                    float a = rec[0], Tj = rec[1], e = rec[2], dx = rec[3], dy = rec[4];
                    float w = a * Tj;
                    float gj = 0.0f;
                    for (int c = 0; c < C; c++) {
                        float fc = feat_at(feat, feat_bytes, C, g, c);
                        gj = fmaf(gf[c], fc, gj);
                        d_feat[g * C + c] += (double)(w * gf[c]);
                    }
                    Sup = fmaf(w, gj, Sup);
                    float oma = 1.0f - a;
                    float dadash = Tj * gj - (S - Sup) / oma + ga * Tend / oma;
                    if (rec[5] != 0.0f) continue;                 /* clamp binds: no gradient */
                    d_alpha[g] += (double)(dadash * e);
                    float dq = dadash * alpha[g] * (-0.5f * e);
                    const float* cn = conic + g * 3;
                    d_conic[g * 3 + 0] += (double)(dq * dx * dx);
                    d_conic[g * 3 + 1] += (double)(dq * dx * dy);
                    d_conic[g * 3 + 2] += (double)(dq * dy * dy);
                    d_mean2[g * 2 + 0] += (double)(dq * -(2.0f * cn[0] * dx + cn[1] * dy));
                    d_mean2[g * 2 + 1] += (double)(dq * -(cn[1] * dx + 2.0f * cn[2] * dy));
                }
            }
    }
    free(cg);
    free(ca_);
}
