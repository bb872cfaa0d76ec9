// raster.cu -- a2 projection + cull, a4 depth sort, a3/a5 tile binning (sm_100a).
//
// Pipeline of one ta_rasterize call:
//   k_init          reset the per-call device scalars and look-back status words
//   k_project       EWA projection of every Gaussian, 32-byte splat record,
//                   depth key scattered BY ID so the depth sort sees id order (tie-break by id)
//   k_sort_digits + k_sort_pass x passes: stable LSD radix sort of the depth keys over only the
//                   bits that vary among visible Gaussians (8-bit digits, one-sweep: global digit
//                   histograms up front, one kernel per pass with decoupled look-back)
//   k_bin_count     per-tile (consecutive depth ranks) counts of the coarse (32 x 32-pixel) bins
//   k_scan          flat exclusive scan of the bin-major [bins x tiles] counts -> run starts, K
//   k_bin_place     per tile: per-warp cursors, then every (Gaussian, bin) entry appended in rank
//                   order: lists come out ordered by (bin, depth, id) without a sort over K entries
#include "common.cuh"
#include "scan.cuh"
#include "internal.h"
#include "project.cuh"

namespace ta {

// ----------------------------------------------------------------------------- k_init
__global__ void k_init(CallState* __restrict__ cs, unsigned long long* __restrict__ status, int n_status,
                       int64_t n_host, const int64_t* __restrict__ n_dev, uint32_t bin_ranks, uint32_t nbins,
                       const uint32_t* __restrict__ stats) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    for (int k = i; k < n_status; k += gridDim.x * blockDim.x) status[k] = 0ull;
    if (i == 0) {
        const int64_t n = n_host >= 0 ? n_host : *n_dev;
        cs->n = (uint32_t)n;
        cs->K = 0;
        cs->sort_total = 0;
        // visibility statistics: accumulated by k_project, or already computed by the fused front end
        cs->n_visible = stats ? stats[2] : 0u;
        cs->key_or = stats ? stats[0] : 0u;
        cs->key_and = stats ? stats[1] : 0xffffffffu;
        cs->sort_parts = (uint32_t)((n + kSortKeysPerBlock - 1) / kSortKeysPerBlock);
        cs->sort_len = 256u * cs->sort_parts;
        cs->bin_P = (uint32_t)((n + bin_ranks - 1) / bin_ranks);    // rank tiles of this call's n
        if (cs->bin_P == 0) cs->bin_P = 1;
        cs->bin_len = nbins * cs->bin_P + 1;
        for (int k = 0; k < 8; k++) cs->scan_counter[k] = 0u;
        cs->epoch = cs->epoch + 1u == 0u ? 1u : cs->epoch + 1u;   // 0 would match zeroed look-back words
        for (int k = 0; k < 8; k++) cs->work[k] = 0ull;
    }
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) (&cs->digit_hist[0][0])[k] = 0u;
}

// ----------------------------------------------------------------------------- k_project
// Two Gaussians per thread (i and i + 256 of the block's 512), their loads issued before either is
// projected, so each thread keeps two records in flight.
__global__ void __launch_bounds__(256) k_project(const float4* __restrict__ pos_alpha,
                                                 const float4* __restrict__ cov, TargetCam cam,
                                                 RasterConsts rc, CallState* __restrict__ cs,
                                                 uint4* __restrict__ rec, uint32_t* __restrict__ key0,
                                                 uint32_t* __restrict__ val0) {
    __shared__ uint32_t s_or[8], s_and[8], s_cnt[8];
    const uint32_t n = cs->n;
    if (blockIdx.x * 512u >= n) return;                    // whole block past the count (uniform)
    const uint32_t ia = blockIdx.x * 512u + threadIdx.x, ib = ia + 256u;
    float4 paA = make_float4(0.f, 0.f, 0.f, 0.f), c0A = paA, c1A = paA, paB = paA, c0B = paA, c1B = paA;
    if (ia < n) { paA = pos_alpha[ia]; c0A = cov[2 * ia]; c1A = cov[2 * ia + 1]; }
    if (ib < n) { paB = pos_alpha[ib]; c0B = cov[2 * ib]; c1B = cov[2 * ib + 1]; }
    bool visA = false, visB = false;
    uint32_t keyA = kCulledKey, keyB = kCulledKey;
    if (ia < n) project_one(ia, paA, c0A, c1A, cam, rc, rec, key0, val0, visA, keyA);
    if (ib < n) project_one(ib, paB, c0B, c1B, cam, rc, rec, key0, val0, visB, keyB);
    const uint32_t kor = __reduce_or_sync(0xffffffffu, (visA ? keyA : 0u) | (visB ? keyB : 0u));
    const uint32_t kand = __reduce_and_sync(0xffffffffu, (visA ? keyA : 0xffffffffu) & (visB ? keyB : 0xffffffffu));
    const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, visA)) + __popc(__ballot_sync(0xffffffffu, visB));
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
// Stable LSD radix sort of the depth keys (id order in, (depth, id) order out) over only the bits
// that vary among visible keys, 8-bit digits, one-sweep style:
//   k_sort_digits   one read of the keys: the global digit histogram of every pass (cs->digit_hist)
//   k_sort_pass     per pass, one kernel: a block takes the next partition of kSortKeysPerBlock keys
//                   (ticket order), ranks them stably (per-warp ballot multisplit, warps in order),
//                   publishes its per-digit counts and looks back over the earlier partitions for
//                   its per-digit global offsets (decoupled look-back, one thread per digit), then
//                   reorders the keys in shared memory by digit so the global writes are runs.
// Inactive passes (beyond the varying bits) return immediately.
__global__ void __launch_bounds__(256) k_sort_digits(const uint32_t* __restrict__ keys, CallState* __restrict__ cs) {
    __shared__ uint32_t s_h[4][256];
    const int npass = sort_passes(cs);
    const uint32_t n = cs->n;
    if (npass == 0 || blockIdx.x * blockDim.x * 8u >= n) return;
    for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) (&s_h[0][0])[k] = 0u;
    __syncthreads();
    const int shift0 = sort_shift(cs, 0);
    // grid-stride over tiles of 2048 keys, 8 consecutive keys per thread (neighbouring source pixels:
    // similar depths, so the high digits come in runs and are counted run-length, one shared atomic
    // per run); the block's histograms go to global memory once
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8u; i0 < n; i0 += gridDim.x * blockDim.x * 8u) {
        uint32_t key[8];
        if (i0 + 8u <= n) {
            const uint4 a = *reinterpret_cast<const uint4*>(keys + i0), b = *reinterpret_cast<const uint4*>(keys + i0 + 4);
            key[0] = a.x; key[1] = a.y; key[2] = a.z; key[3] = a.w; key[4] = b.x; key[5] = b.y; key[6] = b.z; key[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) key[k] = i0 + k < n ? keys[i0 + k] : 0u;
        }
        const int m = (int)min(8u, n - i0);
        for (int p = 0; p < npass; p++) {
            const int sh = shift0 + 8 * p;
            uint32_t prev = 0xffffffffu, run = 0u;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k < m) {
                    const uint32_t d = (key[k] >> sh) & 255u;
                    if (d != prev) {
                        if (run) atomicAdd(&s_h[p][prev], run);
                        prev = d;
                        run = 0u;
                    }
                    run++;
                }
            }
            if (run) atomicAdd(&s_h[p][prev], run);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < npass * 256; k += blockDim.x) {
        const uint32_t v = (&s_h[0][0])[k];
        if (v) atomicAdd(&cs->digit_hist[k >> 8][k & 255], v);
    }
}

// Exclusive scan of v over the 256 threads of the block (one value per thread); s: 8 words.
__device__ __forceinline__ uint32_t block256_excl(uint32_t v, uint32_t* s) {
    const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s[w] = x;
    __syncthreads();
    uint32_t pre = 0u;
#pragma unroll
    for (int k = 0; k < 8; k++) pre += (uint32_t)k < w ? s[k] : 0u;
    __syncthreads();
    return pre + x - v;
}

// Look-back words: epoch << 32 | flag << 30 | count (flag 1: this partition's count, 2: inclusive
// prefix over partitions 0..p).  The epoch (per call, a device counter advanced by k_init, so graph
// replays advance it too) makes stale words of earlier calls invisible.
constexpr uint64_t kLbAgg = 1ull << 30, kLbInc = 2ull << 30;
constexpr uint32_t kLbMask = (1u << 30) - 1u;

// The last pass also writes the pixel box of every rank (boxes[rank]) for the binning kernels.
__global__ void __launch_bounds__(kSortWarps * 32) k_sort_pass(uint32_t* __restrict__ keys_a, uint32_t* __restrict__ keys_b,
                                                               uint32_t* __restrict__ vals_a, uint32_t* __restrict__ vals_b,
                                                               int pass, CallState* __restrict__ cs,
                                                               unsigned long long* __restrict__ lb,
                                                               const uint4* __restrict__ rec, uint2* __restrict__ boxes) {
    static_assert(kSortWarps * 32 == 256, "one thread per digit");
    constexpr int kChunks = kSortKeysPerWarp / 32;
    __shared__ uint32_t s_off[kSortWarps][256];        // per-warp digit counts -> per-warp offsets
    __shared__ uint32_t s_loc[256], s_gbase[256], s_scan[8], s_part;
    __shared__ uint32_t s_key[kSortKeysPerBlock], s_val[kSortKeysPerBlock];
    const int npass = sort_passes(cs);
    if (pass >= npass) return;
    const bool last = pass == npass - 1;
    const uint32_t parts = cs->sort_parts;
    if (blockIdx.x >= parts) return;
    if (threadIdx.x == 0) s_part = atomicAdd(&cs->scan_counter[pass], 1u);
    const uint32_t* sk = (pass & 1) ? keys_b : keys_a;
    const uint32_t* sv = (pass & 1) ? vals_b : vals_a;
    uint32_t* dk = (pass & 1) ? keys_a : keys_b;
    uint32_t* dv = (pass & 1) ? vals_a : vals_b;
    const int shift = sort_shift(cs, pass);
    const uint32_t n = cs->n;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    for (int k = threadIdx.x; k < kSortWarps * 256; k += blockDim.x) (&s_off[0][0])[k] = 0u;
    __syncthreads();
    const uint32_t part = s_part;
    uint32_t* cnt = s_off[warp];
    const uint32_t lt = lanemask_lt();
    const uint32_t b0 = part * kSortKeysPerBlock;
    const uint32_t b = b0 + warp * kSortKeysPerWarp;
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
    const uint32_t d = threadIdx.x;                    // ---- one thread per digit from here
    uint32_t tot = 0u;
#pragma unroll
    for (int w = 0; w < kSortWarps; w++) {             // warps in order within the partition
        const uint32_t c = s_off[w][d];
        s_off[w][d] = tot;
        tot += c;
    }
    unsigned long long* my = lb + (size_t)part * 256 + d;
    const uint32_t epoch = cs->epoch;                  // per call, advanced by k_init on the device
    const unsigned long long ep = (unsigned long long)epoch << 32;
    if (part == 0) *(volatile unsigned long long*)my = ep | kLbInc | tot;
    else *(volatile unsigned long long*)my = ep | kLbAgg | tot;
    const uint32_t loc = block256_excl(tot, s_scan);                              // digit start in the block
    const uint32_t gex = block256_excl(cs->digit_hist[pass][d], s_scan);          // digit start overall
    uint32_t excl = 0u;
    if (part > 0) {                  // decoupled look-back over partitions part-1, part-2, ... 8 at a time
        constexpr int kWin = 8;
        uint32_t q = part;                             // partitions q..part-1 are accounted for
        bool done = false;
        while (!done) {
            unsigned long long w[kWin];
#pragma unroll
            for (int j = 0; j < kWin; j++)
                w[j] = (uint32_t)j < q ? *(volatile unsigned long long*)(lb + (size_t)(q - 1 - j) * 256 + d)
                                       : (ep | kLbInc);
#pragma unroll
            for (int j = 0; j < kWin; j++) {
                if (done) break;
                if ((w[j] >> 32) != epoch) break;      // not published yet: retry from here
                excl += (uint32_t)w[j] & kLbMask;
                q--;
                if (w[j] & kLbInc) done = true;
            }
        }
        *(volatile unsigned long long*)my = ep | kLbInc | (excl + tot);
    }
    s_loc[d] = loc;
    s_gbase[d] = gex + excl;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kChunks; k++) {                // reorder by digit in shared memory
        if (b + k * 32 + lane < n) {
            const uint32_t dd = (key[k] >> shift) & 255u;
            const uint32_t lp = s_loc[dd] + cnt[dd] + rank[k];
            s_key[lp] = key[k];
            s_val[lp] = val[k];
        }
    }
    __syncthreads();
    const uint32_t m = n - b0 < (uint32_t)kSortKeysPerBlock ? n - b0 : (uint32_t)kSortKeysPerBlock;
    constexpr int kIt = kSortKeysPerBlock / (kSortWarps * 32);
    uint2 bq[kIt];                                     // last pass: every pixel box gathered up front
    if (last) {
#pragma unroll
        for (int u = 0; u < kIt; u++) {
            const uint32_t i = threadIdx.x + u * (kSortWarps * 32);
            if (i < m) {
                const uint4 q = rec[2 * s_val[i] + 1];
                bq[u] = make_uint2(q.z, q.w);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kIt; u++) {                    // digit runs -> consecutive addresses
        const uint32_t i = threadIdx.x + u * (kSortWarps * 32);
        if (i < m) {
            const uint32_t k = s_key[i], v = s_val[i];
            const uint32_t dd = (k >> shift) & 255u;
            const uint32_t pos = s_gbase[dd] + (i - s_loc[dd]);
            dk[pos] = k;
            dv[pos] = v;
            if (last) boxes[pos] = bq[u];
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
    constexpr int kIn = 8;                                  // boxes in flight per thread
    for (uint32_t r = tile * R + threadIdx.x; r < r1; r += kIn * blockDim.x) {
        uint2 bx[kIn];
#pragma unroll
        for (int u = 0; u < kIn; u++) {
            const uint32_t rr = r + u * blockDim.x;
            bx[u] = rr < r1 ? boxes[rr] : make_uint2(kEmptyRect, kEmptyRect);
        }
#pragma unroll
        for (int u = 0; u < kIn; u++) count_box(s_h, bx[u], bg);
    }
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
    {
        uint2 bx[kBinRanksPerWarp / 32];                  // all of this lane's boxes in flight at once
#pragma unroll
        for (int u = 0; u < kBinRanksPerWarp / 32; u++) {
            const uint32_t r = wr0 + lane + 32u * u;
            bx[u] = r < wr1 ? boxes[r] : make_uint2(kEmptyRect, kEmptyRect);
        }
#pragma unroll
        for (int u = 0; u < kBinRanksPerWarp / 32; u++) count_box(run, bx[u], bg);
    }
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
    // the next step's box and index are loaded while this step places its entries
    uint2 nb = make_uint2(kEmptyRect, kEmptyRect);
    uint32_t nidx = 0u;
    if (wr0 + lane < wr1) { nb = boxes[wr0 + lane]; nidx = sorted[wr0 + lane]; }
    for (uint32_t r0 = wr0; r0 < wr1; r0 += 32) {
        const uint32_t r = r0 + lane;
        const uint2 pb = nb;
        const uint32_t idx = nidx;
        nb = make_uint2(kEmptyRect, kEmptyRect);
        if (r + 32 < wr1) { nb = boxes[r + 32]; nidx = sorted[r + 32]; }
        int x0 = 1, x1 = 0, y0 = 1, y1 = 0;
        bool ok = false;
        if (r < wr1) ok = box_bins(pb, bg.shift, &x0, &x1, &y0, &y1);
        // compositing tiles covered by the pixel box: each list entry carries, above the index, the
        // rectangle of its coarse bin's tiles the box covers (read by k_tile_split)
        const int ts = bg.ts;
        const int tx0 = (int)(pb.x & 0xffff) >> ts, tx1 = (int)(pb.x >> 16) >> ts;
        const int ty0 = (int)(pb.y & 0xffff) >> ts, ty1 = (int)(pb.y >> 16) >> ts;
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
                const int sb = bg.shift - ts, qm = (1 << sb) - 1;
                const int cx = (x0 + xi) << sb, cy = (y0 + yi) << sb;
                uint32_t rect;
                if (sb == 1) {                               // 2 x 2 tiles: the tile mask itself
                    // inside the box's bin range only the first / last bin column (row) can miss a tile
                    const uint32_t mx = 3u & ~((cx < tx0) ? 1u : 0u) & ~((cx + 1 > tx1) ? 2u : 0u);
                    const uint32_t my = 3u & ~((cy < ty0) ? 1u : 0u) & ~((cy + 1 > ty1) ? 2u : 0u);
                    rect = (mx * (my & 1u)) | ((mx << 2) * (my >> 1));
                } else {                                     // 4 x 4 tiles: the bin-local tile rectangle
                    rect = (uint32_t)max(tx0 - cx, 0) | ((uint32_t)min(tx1 - cx, qm) << sb) |
                           ((uint32_t)max(ty0 - cy, 0) << (2 * sb)) | ((uint32_t)min(ty1 - cy, qm) << (3 * sb));
                }
                if (pos < cap32) list[pos] = idx | (rect << entry_idx_bits(sb));
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
