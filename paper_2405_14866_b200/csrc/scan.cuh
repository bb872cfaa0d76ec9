// scan.cuh -- single-pass exclusive prefix sum of uint32 (decoupled look-back).
//
// Used for the [bins x partitions] offset matrices of the depth sort and of the tile binning
// (both laid out bin-major, so one flat exclusive scan yields every partition's bin offset)
// and for the unprojection's compaction offsets.  Blocks take tiles in arrival order from an
// atomic counter (forward progress of the look-back chain); tile status words pack a 2-bit
// flag with a 62-bit running value.
#pragma once
#include "common.cuh"

namespace ta {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

// Block-wide exclusive scan of one u64 per thread; returns the exclusive prefix, *total = sum.
__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v,
                                                                  unsigned long long* total,
                                                                  unsigned long long* s_warp) {
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    if (warp == 0) {
        unsigned long long w = lane < (uint32_t)nw ? s_warp[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= (uint32_t)o) w += y;
        }
        if (lane < (uint32_t)nw) s_warp[lane] = w;   // inclusive per warp
    }
    __syncthreads();
    const unsigned long long warp_excl = warp ? s_warp[warp - 1] : 0ull;
    *total = s_warp[nw - 1];
    __syncthreads();
    return warp_excl + x - v;
}

// Look-back (warp 0, 32 predecessors per step): publishes this tile's aggregate, sums the
// aggregates of earlier tiles until one with an inclusive prefix is found, publishes the
// inclusive prefix and returns the exclusive prefix to the whole block (broadcast via smem).
__device__ __forceinline__ unsigned long long lookback_prefix(unsigned long long* status, uint32_t tile,
                                                              unsigned long long block_total,
                                                              unsigned long long* s_bcast) {
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        unsigned long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_release_u64(&status[0], kFlagInc | block_total);
        } else {
            if (lane == 0) st_relaxed_u64(&status[tile], kFlagAgg | block_total);
            int p = (int)tile - 1 - (int)lane;
            while (true) {
                unsigned long long s = kFlagInc;       // before tile 0: inclusive prefix 0
                if (p >= 0) {
                    do { s = ld_acquire_u64(&status[p]); } while ((s >> 62) == 0);
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, (s & kFlagInc) != 0);
                unsigned long long v = s & kValMask;
                if (inc) {
                    const int f = __ffs(inc) - 1;      // nearest predecessor with an inclusive prefix
                    if ((int)lane > f) v = 0;
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (inc) break;
                p -= 32;
            }
            if (lane == 0) st_release_u64(&status[tile], kFlagInc | (prefix + block_total));
        }
        if (lane == 0) *s_bcast = prefix;
    }
    __syncthreads();
    return *s_bcast;
}

// In-place exclusive scan of data[0 .. *len) ; *total = sum.  status[] must be zero and
// *counter zero before the launch (k_init does it).  Grid: >= ceil(len / kScanTile) blocks.
__global__ void __launch_bounds__(kScanThreads) k_scan_excl_u32(uint32_t* __restrict__ data,
                                                                const uint32_t* __restrict__ len_ptr, uint32_t len_host,
                                                                unsigned long long* __restrict__ status,
                                                                uint32_t* __restrict__ counter,
                                                                unsigned long long* __restrict__ total) {
    __shared__ unsigned long long s_warp[kScanThreads / 32];
    __shared__ unsigned long long s_bcast;
    __shared__ uint32_t s_tile;
    const uint32_t len = len_ptr ? *len_ptr : len_host;
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = (uint64_t)tile * kScanTile;
    if (base >= len) {
        if (tile == 0 && threadIdx.x == 0) *total = 0;
        return;
    }
    const uint64_t i0 = base + (uint64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    if (i0 + kScanItems <= len) {
        const uint4 a = *reinterpret_cast<const uint4*>(data + i0);
        const uint4 b = *reinterpret_cast<const uint4*>(data + i0 + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; k++) v[k] = (i0 + k < len) ? data[i0 + k] : 0u;
    }
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) sum += v[k];
    unsigned long long btotal;
    const unsigned long long texcl = block_excl_scan_u64(sum, &btotal, s_warp);
    const unsigned long long prefix = lookback_prefix(status, tile, btotal, &s_bcast);
    unsigned long long run = prefix + texcl;
    uint32_t o[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) { o[k] = (uint32_t)run; run += v[k]; }
    if (i0 + kScanItems <= len) {
        *reinterpret_cast<uint4*>(data + i0) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(data + i0 + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; k++)
            if (i0 + k < len) data[i0 + k] = o[k];
    }
    if (base + kScanTile >= len && threadIdx.x == 0) *total = prefix + btotal;
}

}  // namespace ta
