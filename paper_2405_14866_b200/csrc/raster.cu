// raster.cu -- a2 projection + cull, a4 depth sort, a3/a5 tile binning (sm_100a).
//
// Pipeline of one ta_rasterize call:
//   k_init          reset the per-call device scalars and look-back status words
//   k_project       EWA projection of every Gaussian, 32-byte splat record,
//                   depth key scattered BY ID so the depth sort sees id order (tie-break by id)
//   k_sort_hist / k_scan / k_sort_scatter   x passes: stable LSD radix sort of the depth keys over
//                   only the bits that vary among visible Gaussians (8-bit digits, per-warp
//                   partitions, warp-synchronous stable ranking with match.any)
//   k_bin_count     per-warp tile histograms of a contiguous depth-rank range, via 2-D
//                   difference arrays (4 updates per Gaussian instead of one per tile)
//   k_scan          over the tile-major [T x P] count matrix -> every (tile, warp) list offset,
//                   tile ranges and the entry total K in one flat exclusive scan
//   k_bin_place     each warp walks its depth-rank range in order and appends the Gaussian's
//                   array index to every covered tile's list: lists come out ordered by
//                   (tile, depth, id) without a global sort over the K entries
#include "common.cuh"
#include "scan.cuh"
#include "internal.h"

namespace ta {

// ----------------------------------------------------------------------------- k_init
__global__ void k_init(CallState* __restrict__ cs, unsigned long long* __restrict__ status, int n_status,
                       int64_t n_host, const int64_t* __restrict__ n_dev, uint32_t bin_len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = i; k < n_status; k += gridDim.x * blockDim.x) status[k] = 0ull;
    if (i == 0) {
        const int64_t n = n_host >= 0 ? n_host : *n_dev;
        cs->n = (uint32_t)n;
        cs->K = 0;
        cs->sort_total = 0;
        cs->n_visible = 0;
        cs->key_or = 0u;
        cs->key_and = 0xffffffffu;
        cs->sort_parts = (uint32_t)((n + kSortKeysPerBlock - 1) / kSortKeysPerBlock);
        cs->sort_len = 256u * cs->sort_parts;
        cs->bin_len = bin_len;
        for (int k = 0; k < 8; k++) cs->scan_counter[k] = 0u;
        for (int k = 0; k < 8; k++) cs->work[k] = 0ull;
    }
}

// ----------------------------------------------------------------------------- k_project
// Normative sequence of DESIGN.md a2 (mirrors nothing: the oracle is separate C code).
__global__ void __launch_bounds__(256) k_project(const float4* __restrict__ pos_alpha,
                                                 const float4* __restrict__ cov, TargetCam cam,
                                                 RasterConsts rc, CallState* __restrict__ cs,
                                                 uint4* __restrict__ rec, uint32_t* __restrict__ key0,
                                                 uint32_t* __restrict__ val0) {
    __shared__ uint32_t s_or[8], s_and[8], s_cnt[8];
    const uint32_t n = cs->n;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool vis = false;
    uint32_t key = kCulledKey;
    if (i < n) {
        const float4 pa = pos_alpha[i];
        const float4 c0 = cov[2 * i], c1 = cov[2 * i + 1];
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
    const uint32_t kor = __reduce_or_sync(0xffffffffu, vis ? key : 0u);
    const uint32_t kand = __reduce_and_sync(0xffffffffu, vis ? key : 0xffffffffu);
    const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, vis));
    const uint32_t w = threadIdx.x >> 5;
    if (lane_id() == 0) { s_or[w] = kor; s_and[w] = kand; s_cnt[w] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t o = 0, a = 0xffffffffu, c = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) { o |= s_or[k]; a &= s_and[k]; c += s_cnt[k]; }
        if (c) {
            atomicOr(&cs->key_or, o);
            atomicAnd(&cs->key_and, a);
            atomicAdd(&cs->n_visible, c);
        }
    }
}

// ----------------------------------------------------------------------------- depth sort
// Pass `pass` sorts by 8 bits starting at sort_shift(); keys/vals ping-pong a -> b -> a ...
// Inactive passes (beyond the varying bits) return immediately.  A block owns kSortKeysPerBlock
// consecutive keys, each warp kSortKeysPerWarp of them in order; warps rank their keys stably
// (match.any per 32-key chunk, per-warp digit counters), the block combines warps in order.
__global__ void __launch_bounds__(kSortWarps * 32) k_sort_hist(const uint32_t* __restrict__ keys_a,
                                                               const uint32_t* __restrict__ keys_b, int pass,
                                                               const CallState* __restrict__ cs,
                                                               uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_cnt[kSortWarps][256];
    if (pass >= sort_passes(cs)) return;
    const uint32_t parts = cs->sort_parts;
    if (blockIdx.x >= parts) return;
    const uint32_t* src = (pass & 1) ? keys_b : keys_a;
    const int shift = sort_shift(cs, pass);
    const uint32_t n = cs->n;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    for (int k = threadIdx.x; k < kSortWarps * 256; k += blockDim.x) (&s_cnt[0][0])[k] = 0u;
    __syncthreads();
    uint32_t* cnt = s_cnt[warp];
    constexpr int kChunks = kSortKeysPerWarp / 32;
    const uint32_t b = blockIdx.x * kSortKeysPerBlock + warp * kSortKeysPerWarp;
    uint32_t key[kChunks];
#pragma unroll
    for (int k = 0; k < kChunks; k++) {          // all loads in flight before any ranking
        const uint32_t idx = b + k * 32 + lane;
        key[k] = idx < n ? src[idx] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kChunks; k++) {
        const bool ok = b + k * 32 + lane < n;
        const uint32_t d = ok ? (key[k] >> shift) & 255u : 0u;
        const uint32_t peers = peers8(d, __ballot_sync(0xffffffffu, ok));
        if (ok && lane == (uint32_t)(__ffs(peers) - 1)) cnt[d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    const uint32_t d = threadIdx.x;
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; w++) sum += s_cnt[w][d];
    hist[(size_t)d * parts + blockIdx.x] = sum;
}

__global__ void __launch_bounds__(kSortWarps * 32) k_sort_scatter(uint32_t* __restrict__ keys_a, uint32_t* __restrict__ keys_b,
                                                                  uint32_t* __restrict__ vals_a, uint32_t* __restrict__ vals_b,
                                                                  int pass, const CallState* __restrict__ cs,
                                                                  const uint32_t* __restrict__ offs) {
    constexpr int kChunks = kSortKeysPerWarp / 32;
    __shared__ uint32_t s_off[kSortWarps][256];
    if (pass >= sort_passes(cs)) return;
    const uint32_t parts = cs->sort_parts;
    if (blockIdx.x >= parts) return;
    const uint32_t* sk = (pass & 1) ? keys_b : keys_a;
    const uint32_t* sv = (pass & 1) ? vals_b : vals_a;
    uint32_t* dk = (pass & 1) ? keys_a : keys_b;
    uint32_t* dv = (pass & 1) ? vals_a : vals_b;
    const int shift = sort_shift(cs, pass);
    const uint32_t n = cs->n;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    for (int k = threadIdx.x; k < kSortWarps * 256; k += blockDim.x) (&s_off[0][0])[k] = 0u;
    __syncthreads();
    uint32_t* cnt = s_off[warp];
    const uint32_t lt = lanemask_lt();
    const uint32_t b = blockIdx.x * kSortKeysPerBlock + warp * kSortKeysPerWarp;
    uint32_t key[kChunks], val[kChunks], rank[kChunks];
#pragma unroll
    for (int k = 0; k < kChunks; k++) {
        const uint32_t idx = b + k * 32 + lane;
        const bool ok = idx < n;
        key[k] = ok ? sk[idx] : 0u;
        val[k] = ok ? sv[idx] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kChunks; k++) {
        const bool ok = b + k * 32 + lane < n;
        const uint32_t d = ok ? (key[k] >> shift) & 255u : 0u;
        const uint32_t peers = peers8(d, __ballot_sync(0xffffffffu, ok));
        const uint32_t base = ok ? cnt[d] : 0u;
        __syncwarp();
        rank[k] = base + __popc(peers & lt);
        if (ok && lane == (uint32_t)(__ffs(peers) - 1)) cnt[d] = base + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // per digit: warps in order after the block's global offset
        const uint32_t d = threadIdx.x;
        uint32_t run = offs[(size_t)d * parts + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) {
            const uint32_t c = s_off[w][d];
            s_off[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kChunks; k++) {
        if (b + k * 32 + lane < n) {
            const uint32_t pos = cnt[(key[k] >> shift) & 255u] + rank[k];
            dk[pos] = key[k];
            dv[pos] = val[k];
        }
    }
}

// ----------------------------------------------------------------------------- binning
__device__ __forceinline__ void rank_range(uint32_t n, uint32_t P, uint32_t p, uint32_t* rb, uint32_t* re) {
    *rb = (uint32_t)(((uint64_t)n * p) / P);
    *re = (uint32_t)(((uint64_t)n * (p + 1)) / P);
}

__device__ __forceinline__ const uint32_t* sorted_vals(const CallState* cs, const uint32_t* vals_a,
                                                       const uint32_t* vals_b) {
    return (sort_passes(cs) & 1) ? vals_b : vals_a;
}

// Pixel boxes in depth-rank order (coalesced input for both binning kernels).
__global__ void __launch_bounds__(256) k_gather_boxes(const uint4* __restrict__ rec, const uint32_t* __restrict__ vals_a,
                                                      const uint32_t* __restrict__ vals_b,
                                                      const CallState* __restrict__ cs, uint2* __restrict__ boxes) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= cs->n) return;
    const uint32_t* sorted = sorted_vals(cs, vals_a, vals_b);
    const uint4 q = rec[2 * sorted[r] + 1];
    boxes[r] = make_uint2(q.z, q.w);
}

// Per-warp tile counts over depth ranks [rb, re): 2-D difference array on a (TY+1) x GW grid
// (GW = (TX+1)|1, odd to spread banks), prefix-summed in place, then written tile-major
// into counts[t * P + p].  The last element counts[T*P] is zeroed (it becomes K after the scan).
__global__ void __launch_bounds__(512) k_bin_count(const uint2* __restrict__ boxes, const CallState* __restrict__ cs,
                                                   BinGeom bg, uint32_t* __restrict__ counts) {
    extern __shared__ int32_t s_grid[];
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int nw = blockDim.x >> 5;
    const int GW = bg.GW, GH = bg.TY + 1, GS = bg.GS;
    int32_t* grid = s_grid + (size_t)warp * GS;
    for (int k = lane; k < GS; k += 32) grid[k] = 0;
    __syncwarp();
    const uint32_t p = blockIdx.x * nw + warp;
    uint32_t rb, re;
    rank_range(cs->n, bg.P, p, &rb, &re);
    uint2 nxt = rb + lane < re ? boxes[rb + lane] : make_uint2(kEmptyRect, kEmptyRect);
    for (uint32_t r0 = rb; r0 < re; r0 += 32) {
        const uint2 bx = nxt;
        nxt = r0 + 32 + lane < re ? boxes[r0 + 32 + lane] : make_uint2(kEmptyRect, kEmptyRect);
        bool ok = r0 + lane < re;
        const uint32_t rx = bx.x, ry = bx.y;
        const int x0 = rx & 0xffff, x1 = rx >> 16, y0 = ry & 0xffff, y1 = ry >> 16;
        ok = ok && x0 <= x1 && y0 <= y1;
        const int sh = bg.shift;
        const int tx0 = x0 >> sh, tx1 = (x1 >> sh) + 1, ty0 = y0 >> sh, ty1 = (y1 >> sh) + 1;
#pragma unroll
        for (int corner = 0; corner < 4; corner++) {
            const int cy = (corner & 2) ? ty1 : ty0;
            const int cx = (corner & 1) ? tx1 : tx0;
            const int sign = (corner == 0 || corner == 3) ? 1 : -1;
            const uint32_t cell = ok ? (uint32_t)(cy * GW + cx) : (0x80000000u | lane);
            const uint32_t peers = __match_any_sync(0xffffffffu, cell);
            if (ok && lane == (uint32_t)(__ffs(peers) - 1)) grid[cell] += sign * __popc(peers);
            __syncwarp();
        }
    }
    // 2-D inclusive prefix: rows, then columns
    for (int row = lane; row < GH; row += 32) {
        int32_t acc = 0;
        int32_t* g = grid + row * GW;
        for (int x = 0; x < GW; x++) { acc += g[x]; g[x] = acc; }
    }
    __syncwarp();
    for (int col = lane; col < GW; col += 32) {
        int32_t acc = 0;
        for (int y = 0; y < GH; y++) { acc += grid[y * GW + col]; grid[y * GW + col] = acc; }
    }
    __syncthreads();
    const int T = bg.TX * bg.TY;
    for (int k = threadIdx.x; k < T * nw; k += blockDim.x) {
        const int t = k / nw, w = k % nw;
        const uint32_t pp = blockIdx.x * nw + w;
        const int ty = t / bg.TX, tx = t - ty * bg.TX;
        counts[(size_t)t * bg.P + pp] = (uint32_t)s_grid[(size_t)w * GS + ty * GW + tx];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) counts[(size_t)T * bg.P] = 0u;
}

// Each warp appends its depth-rank range to the tile lists, in rank order.  32 consecutive
// (Gaussian, tile) entries per step; same-tile entries inside a step are ordered by lane with
// match.any, so each list stays ordered by (depth, id).
__global__ void __launch_bounds__(512) k_bin_place(const uint2* __restrict__ boxes, const uint32_t* __restrict__ vals_a,
                                                   const uint32_t* __restrict__ vals_b,
                                                   CallState* __restrict__ cs, BinGeom bg,
                                                   const uint32_t* __restrict__ offs, uint32_t* __restrict__ list,
                                                   uint64_t list_cap) {
    extern __shared__ uint32_t s_run[];
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int nw = blockDim.x >> 5;
    const int T = bg.TX * bg.TY;
    for (int k = threadIdx.x; k < T * nw; k += blockDim.x) {
        const int t = k / nw, w = k % nw;
        s_run[(size_t)w * T + t] = offs[(size_t)t * bg.P + blockIdx.x * nw + w];
    }
    __syncthreads();
    uint32_t* run = s_run + (size_t)warp * T;
    const uint32_t* sorted = sorted_vals(cs, vals_a, vals_b);
    const uint32_t p = blockIdx.x * nw + warp;
    const uint32_t lt = lanemask_lt();
    uint32_t rb, re;
    rank_range(cs->n, bg.P, p, &rb, &re);
    bool overflow = false;
    uint32_t nidx = rb + lane < re ? sorted[rb + lane] : 0u;
    uint2 nbx = rb + lane < re ? boxes[rb + lane] : make_uint2(kEmptyRect, kEmptyRect);
    for (uint32_t r0 = rb; r0 < re; r0 += 32) {
        const uint32_t idx = nidx;
        const uint32_t rx = nbx.x, ry = nbx.y;
        const uint32_t rn = r0 + 32 + lane;
        nidx = rn < re ? sorted[rn] : 0u;
        nbx = rn < re ? boxes[rn] : make_uint2(kEmptyRect, kEmptyRect);
        const int x0 = rx & 0xffff, x1 = rx >> 16, y0 = ry & 0xffff, y1 = ry >> 16;
        const bool ok = x0 <= x1 && y0 <= y1;
        const int sh = bg.shift;
        const int tx0 = x0 >> sh, ty0 = y0 >> sh;
        const int tw = ok ? (x1 >> sh) - tx0 + 1 : 1;
        const uint32_t cnt = ok ? (uint32_t)(tw * ((y1 >> sh) - ty0 + 1)) : 0u;
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        const uint32_t excl = incl - cnt;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t org = (uint32_t)tx0 | ((uint32_t)ty0 << 16);
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t j = e0 + lane;
            const bool valid = j < total;
            // largest window lane k with excl_k <= j (always a lane with cnt_k > 0)
            int k = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                const uint32_t ex = __shfl_sync(0xffffffffu, excl, k + s);
                if (ex <= j) k += s;
            }
            const uint32_t ex_k = __shfl_sync(0xffffffffu, excl, k);
            const uint32_t idx_k = __shfl_sync(0xffffffffu, idx, k);
            const uint32_t org_k = __shfl_sync(0xffffffffu, org, k);
            const int tw_k = __shfl_sync(0xffffffffu, tw, k);
            const int m = (int)(j - ex_k);
            int row = (int)__fmul_rz((float)m + 0.5f, __frcp_rn((float)tw_k));
            if (row * tw_k > m) row--;
            if ((row + 1) * tw_k <= m) row++;
            const int col = m - row * tw_k;
            const uint32_t t = (uint32_t)(((int)(org_k >> 16) + row) * bg.TX + (int)(org_k & 0xffff) + col);
            const uint32_t key = valid ? t : (0x80000000u | lane);
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const uint32_t base = valid ? run[t] : 0u;
            __syncwarp();
            if (valid) {
                const uint32_t pos = base + __popc(peers & lt);
                if (pos < list_cap) list[pos] = idx_k;
                else overflow = true;
                if (lane == (uint32_t)(__ffs(peers) - 1)) run[t] = base + __popc(peers);
            }
            __syncwarp();
        }
    }
    if (overflow) atomicOr(&cs->overflow, 1u);
}

}  // namespace ta

namespace ta {
void launch_scan(uint32_t* data, const uint32_t* len_ptr, uint32_t len_max, unsigned long long* status,
                 uint32_t* counter, unsigned long long* total, cudaStream_t st) {
    const uint32_t blocks = len_max / kScanTile + 1;
    k_scan_excl_u32<<<blocks, kScanThreads, 0, st>>>(data, len_ptr, len_max, status, counter, total);
}
}  // namespace ta
