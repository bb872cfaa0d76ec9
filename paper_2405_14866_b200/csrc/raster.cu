// raster.cu -- a2 projection + cull, a4 depth sort, a3/a5 tile binning (sm_100a).
//
// Pipeline of one ta_rasterize call:
//   k_init          reset the per-call device scalars and look-back status words
//   k_project       EWA projection of every Gaussian, 32-byte splat record,
//                   depth key scattered BY ID so the depth sort sees id order (tie-break by id)
//   k_sort_hist / k_scan / k_sort_scatter   x passes: stable LSD radix sort of the depth keys over
//                   only the bits that vary among visible Gaussians (8-bit digits, per-warp
//                   partitions, warp-synchronous stable ranking with ballot multisplit)
//   k_bin_count     per-tile (consecutive depth ranks) counts of the coarse (32 x 32-pixel) bins
//   k_scan          flat exclusive scan of the bin-major [bins x tiles] counts -> run starts, K
//   k_bin_place     per tile: per-warp cursors, then every (Gaussian, bin) entry appended in rank
//                   order: lists come out ordered by (bin, depth, id) without a sort over K entries
#include "common.cuh"
#include "scan.cuh"
#include "internal.h"

namespace ta {

// ----------------------------------------------------------------------------- k_init
__global__ void k_init(CallState* __restrict__ cs, unsigned long long* __restrict__ status, int n_status,
                       int64_t n_host, const int64_t* __restrict__ n_dev, uint32_t bin_ranks, uint32_t nbins) {
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
        cs->bin_P = (uint32_t)((n + bin_ranks - 1) / bin_ranks);    // rank tiles of this call's n
        if (cs->bin_P == 0) cs->bin_P = 1;
        cs->bin_len = nbins * cs->bin_P + 1;
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
    if (blockIdx.x * blockDim.x >= n) return;              // whole block past the count (uniform)
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
// (ballot multisplit per 32-key chunk, per-warp digit counters), the block combines warps in order.
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

// The last pass also writes the pixel box of every rank (boxes[rank]) for the binning kernels.
__global__ void __launch_bounds__(kSortWarps * 32) k_sort_scatter(uint32_t* __restrict__ keys_a, uint32_t* __restrict__ keys_b,
                                                                  uint32_t* __restrict__ vals_a, uint32_t* __restrict__ vals_b,
                                                                  int pass, const CallState* __restrict__ cs,
                                                                  const uint32_t* __restrict__ offs,
                                                                  const uint4* __restrict__ rec, uint2* __restrict__ boxes) {
    constexpr int kChunks = kSortKeysPerWarp / 32;
    __shared__ uint32_t s_off[kSortWarps][256];
    const int npass = sort_passes(cs);
    if (pass >= npass) return;
    const bool last = pass == npass - 1;
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
            if (last) {
                const uint4 q = rec[2 * val[k] + 1];
                boxes[pos] = make_uint2(q.z, q.w);
            }
        }
    }
}

// ----------------------------------------------------------------------------- binning
// Coarse bins are (1 << shift)-pixel squares.  The per-bin lists hold the array index of every
// visible Gaussian whose pixel box overlaps the bin, in depth-rank order: a stable counting sort
// of the (Gaussian, bin) entries by bin, the entries being generated on the fly from the
// rank-ordered boxes.  The ranks are cut into P tiles of R = nw * 256 consecutive ranks:
//   k_bin_count  per-tile bin counts -> counts[bin * P + tile] (bin-major)
//   (scan)       one flat exclusive scan: the start of every (bin, tile) run, K = entries
//   k_bin_place  per tile: per-warp bin counts, exclusive scan over the warps (cursors), then each
//                warp re-walks its ranks and appends every entry at its cursor: lists come out in
//                (bin, depth, id) order.  List of bin b = [offs[b * P], offs[(b + 1) * P]).
constexpr int kBinRanksPerWarp = 256;

// Pixel boxes in depth-rank order; only used when the depth sort ran no pass (otherwise the last
// scatter pass writes them).
__global__ void __launch_bounds__(256) k_gather_boxes(const uint4* __restrict__ rec, const uint32_t* __restrict__ vals_a,
                                                      const uint32_t* __restrict__ vals_b,
                                                      const CallState* __restrict__ cs, uint2* __restrict__ boxes) {
    if (sort_passes(cs) > 0) return;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < cs->n; r += gridDim.x * blockDim.x) {
        const uint4 q = rec[2 * vals_a[r] + 1];
        boxes[r] = make_uint2(q.z, q.w);
    }
}

__device__ __forceinline__ bool box_bins(uint2 bx, int sh, int* bx0, int* bx1, int* by0, int* by1) {
    const int x0 = bx.x & 0xffff, x1 = bx.x >> 16, y0 = bx.y & 0xffff, y1 = bx.y >> 16;
    *bx0 = x0 >> sh;
    *bx1 = x1 >> sh;
    *by0 = y0 >> sh;
    *by1 = y1 >> sh;
    return x0 <= x1 && y0 <= y1;
}

// Adds 1 to cnt[bin] for every bin of the box (row-major walk of the bin rectangle).
__device__ __forceinline__ void count_box(uint32_t* cnt, uint2 box, const BinGeom& bg) {
    int x0, x1, y0, y1;
    if (!box_bins(box, bg.shift, &x0, &x1, &y0, &y1)) return;
    for (int y = y0; y <= y1; y++)
        for (int x = x0; x <= x1; x++) atomicAdd(&cnt[y * bg.TX + x], 1u);
}

__global__ void __launch_bounds__(256) k_bin_count(const uint2* __restrict__ boxes, const CallState* __restrict__ cs,
                                                   BinGeom bg, uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t s_h[];
    const int NB = bg.TX * bg.TY;
    const uint32_t tile = blockIdx.x, P = cs->bin_P;
    if (tile >= P) return;                                  // grid sized for the capacity
    for (int k = threadIdx.x; k < NB; k += blockDim.x) s_h[k] = 0u;
    if (tile == 0 && threadIdx.x == 0) counts[(size_t)NB * P] = 0u;
    __syncthreads();
    const uint32_t n = cs->n;
    const uint32_t R = (uint32_t)bg.nw * kBinRanksPerWarp;
    const uint32_t r1 = min(n, (tile + 1) * R);
    for (uint32_t r = tile * R + threadIdx.x; r < r1; r += blockDim.x) count_box(s_h, boxes[r], bg);
    __syncthreads();
    for (int k = threadIdx.x; k < NB; k += blockDim.x) counts[(size_t)k * P + tile] = s_h[k];
}

__global__ void __launch_bounds__(256) k_bin_place(const uint2* __restrict__ boxes, const uint32_t* __restrict__ vals_a,
                                                   const uint32_t* __restrict__ vals_b, CallState* __restrict__ cs,
                                                   BinGeom bg, const uint32_t* __restrict__ offs,
                                                   uint32_t* __restrict__ list, uint64_t list_cap) {
    extern __shared__ uint32_t s_cnt[];          // [nw][NB] counts, then write cursors; [nw][NB] lane masks
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int nw = blockDim.x >> 5;
    const int NB = bg.TX * bg.TY;
    const uint32_t n = cs->n;
    const uint32_t tile = blockIdx.x, P = cs->bin_P;
    if (tile >= P) return;
    for (int k = threadIdx.x; k < (nw * NB) / 2; k += blockDim.x)       // 2 nw NB words (NB even or not)
        reinterpret_cast<uint4*>(s_cnt)[k] = make_uint4(0u, 0u, 0u, 0u);
    if (threadIdx.x == 0 && (nw * NB) % 2) { s_cnt[2 * nw * NB - 2] = 0u; s_cnt[2 * nw * NB - 1] = 0u; }
    __syncthreads();
    const uint32_t R = (uint32_t)nw * kBinRanksPerWarp;
    if ((uint64_t)tile * R >= n) return;
    const uint32_t* sorted = (sort_passes(cs) & 1) ? vals_b : vals_a;
    const uint32_t wr0 = tile * R + warp * kBinRanksPerWarp;
    const uint32_t wr1 = min(n, wr0 + kBinRanksPerWarp);
    uint32_t* run = s_cnt + (size_t)warp * NB;
    // ---- per-warp bin counts of the warp's ranks
    for (uint32_t r = wr0 + lane; r < wr1; r += 32) count_box(run, boxes[r], bg);
    __syncthreads();
    // ---- per bin: cursors = start of the (bin, tile) run + entries of the earlier warps
    for (int b = threadIdx.x; b < NB; b += blockDim.x) {
        uint32_t cur = offs[(size_t)b * P + tile];
        for (int w = 0; w < nw; w++) {
            const uint32_t c = s_cnt[w * NB + b];
            s_cnt[w * NB + b] = cur;
            cur += c;
        }
    }
    __syncthreads();
    // ---- phase B: each warp re-walks its ranks in order, one Gaussian per lane, looping over the
    //      bins of its box.  Same-bin entries of one 32-Gaussian step are ranked by lane through a
    //      per-warp lane bitmask per bin (set, read, then cleared by the lowest lane of the mask).
    const uint32_t mbase = (uint32_t)(nw + warp) * NB, rbase = warp * (uint32_t)NB;
    const uint32_t lt = lanemask_lt(), bit = 1u << lane;
    const uint32_t cap32 = (uint32_t)min(list_cap, (uint64_t)0xffffffffu);
    uint32_t overflow = 0u;
    for (uint32_t r0 = wr0; r0 < wr1; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint32_t idx = 0u;
        int x0 = 1, x1 = 0, y0 = 1, y1 = 0;
        bool ok = false;
        uint2 pb = make_uint2(kEmptyRect, kEmptyRect);
        if (r < wr1) {
            pb = boxes[r];
            ok = box_bins(pb, bg.shift, &x0, &x1, &y0, &y1);
            idx = sorted[r];
        }
        // 16 x 16 tiles covered by the pixel box: the list entry carries, above the index, which of the
        // 2 x 2 tiles of its coarse bin the box covers (read by k_tile_split)
        const int tx0 = (int)(pb.x & 0xffff) >> 4, tx1 = (int)(pb.x >> 16) >> 4;
        const int ty0 = (int)(pb.y & 0xffff) >> 4, ty1 = (int)(pb.y >> 16) >> 4;
        const int tw = x1 - x0 + 1;
        const int cnt = ok ? tw * (y1 - y0 + 1) : 0;
        const int maxc = __reduce_max_sync(0xffffffffu, cnt);
        const uint32_t t0 = (uint32_t)(y0 * bg.TX + x0), stride = (uint32_t)(bg.TX - tw);
#pragma unroll 1
        for (int i = 0, xi = 0, t = t0; i < maxc; i++) {
            if (i < cnt) {
                atomicOr(&s_cnt[mbase + t], bit);
                t++;
                if (++xi == tw) { xi = 0; t += stride; }
            }
        }
        __syncwarp();
#pragma unroll 1
        for (int i = 0, xi = 0, yi = 0, t = t0; i < maxc; i++) {
            if (i < cnt) {
                const uint32_t pos = s_cnt[rbase + t] + __popc(s_cnt[mbase + t] & lt);
                const int cx = 2 * (x0 + xi), cy = 2 * (y0 + yi);
                const uint32_t mx = (uint32_t)(cx >= tx0 && cx <= tx1) | ((uint32_t)(cx + 1 >= tx0 && cx + 1 <= tx1) << 1);
                const uint32_t my = (uint32_t)(cy >= ty0 && cy <= ty1) | ((uint32_t)(cy + 1 >= ty0 && cy + 1 <= ty1) << 1);
                const uint32_t tm = ((my & 1u) ? mx : 0u) | ((my & 2u) ? (mx << 2) : 0u);
                if (pos < cap32) list[pos] = idx | (tm << kListIdxBits);
                else overflow = 1u;
                t++;
                if (++xi == tw) { xi = 0; yi++; t += stride; }
            }
        }
        __syncwarp();
#pragma unroll 1
        for (int i = 0, xi = 0, t = t0; i < maxc; i++) {
            if (i < cnt) {
                const uint32_t m = s_cnt[mbase + t];
                if ((m & bit) && !(m & lt)) {          // lowest lane of the mask: advance the cursor, clear
                    s_cnt[rbase + t] += __popc(m);
                    s_cnt[mbase + t] = 0u;
                }
                t++;
                if (++xi == tw) { xi = 0; t += stride; }
            }
        }
        __syncwarp();
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
