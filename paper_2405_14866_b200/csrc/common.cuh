// common.cuh -- device-side building blocks shared by the rasterizer kernels (sm_100a).
//
// The fp32 arithmetic here is this library's own implementation of DESIGN.md "Normative
// arithmetic": every rounding step is an explicit __f*_rn intrinsic so nvcc cannot contract
// or reorder it; that is what makes tile lists, depth order and transmittance reproduce the
// CPU oracle bit for bit (the oracle is a separate C file; the two share no code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

namespace ta {

constexpr int kTile = 16;
// Coarse bins are 2^shift-pixel squares of 2^sb x 2^sb compositing tiles of 2^ts pixels (sb = shift - ts):
// 32 x 32-pixel bins for targets up to 1024 pixels on a side, 64 x 64 beyond (api.cu bin_geometry), so
// the bin count stays ~1024; tiles of 8 x 8 pixels (ts = 3) under 32-pixel bins, 16 x 16 (ts = 4)
// otherwise.  A coarse-list entry is the Gaussian's array index in the low 32 - 4 sb bits and, above
// it, the bin's tiles its pixel box covers: for sb = 1 the 4-bit mask of the 2 x 2 tiles (bit
// qy*2+qx), for sb = 2 the bin-local tile rectangle x0 | x1 << 2 | y0 << 4 | y1 << 6.
constexpr int kMaxCoarseShift = 6;
__host__ __device__ constexpr int entry_idx_bits(int sb) { return 32 - 4 * sb; }
constexpr uint32_t kCulledKey = 0xffffffffu;
constexpr uint32_t kEmptyRect = 1u;     // x0 = 1, x1 = 0  -> empty box

// ------------------------------------------------------------------ exact fp32 helpers
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }

// dot3(a, b) = fma(a2, b2, fma(a1, b1, a0*b0))
__device__ __forceinline__ float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return ffma(a2, b2, ffma(a1, b1, fmul(a0, b0)));
}

// DESIGN.md R13 exp_det: exp(x), x <= 0, by a fixed fp32 sequence (nearest-even k, one-constant
// reduction, degree-6 relative minimax polynomial).
__device__ __forceinline__ float exp_det(float x) {
    x = fmaxf(x, -80.0f);
    const float k = fsub(ffma(x, 1.44269502162933349609375f, 12582912.0f), 12582912.0f);   // nearest-even of x*log2e
    const float r = ffma(-k, 0.693147182464599609375f, x);
    float p = 1.3814548728987575e-3f;
    p = ffma(p, r, 8.36869515478611e-3f);
    p = ffma(p, r, 4.166838899254799e-2f);
    p = ffma(p, r, 1.666652113199234e-1f);
    p = ffma(p, r, 4.999999403953552e-1f);
    p = ffma(p, r, 1.0f);
    p = ffma(p, r, 1.0f);
    const float s = __int_as_float(((int)k + 127) << 23);
    return fmul(p, s);
}

// ------------------------------------------------------------------ memory-order helpers
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of the warp whose 8-bit digit equals this lane's (warp multisplit with 8 ballots; no
// match.any, which throttles the MIO pipe).  Lanes outside `valid` never count as peers.
__device__ __forceinline__ uint32_t peers8(uint32_t d, uint32_t valid) {
    uint32_t m = valid;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bal : ~bal;
    }
    return m;
}

// ------------------------------------------------------------------ per-call device state
// One small struct of device scalars, reset by k_init at the start of every rasterize call.
struct CallState {
    unsigned long long K;          // tile entries (written by the bin-offset scan)
    unsigned long long sort_total; // scratch totals of the sort scans
    uint32_t n;                    // Gaussians of this call
    uint32_t n_visible;
    uint32_t key_or, key_and;      // OR / AND of visible depth keys -> varying bit range
    uint32_t sort_parts;           // depth-sort partitions (blocks): ceil(n / kSortKeysPerBlock)
    uint32_t sort_len;             // 256 * sort_parts
    uint32_t bin_len;              // NB * bin_P + 1 (bin-major run starts + the total)
    uint32_t bin_P;                // rank tiles of this call (ceil(n / ranks per tile))
    uint32_t overflow;             // sticky: entries exceeded the list capacity (not reset by k_init)
    uint32_t epoch;                // depth-sort look-back tag of the current call (advanced by k_init)
    uint32_t scan_counter[8];      // tile counters of the look-back scans (one per scan)
    unsigned long long work[8];    // compositor work counters (TA_FLAG_DEBUG_COUNTS only, reset by k_init)
    uint32_t digit_hist[4][256];   // depth sort: global digit histogram of each pass (k_sort_digits)
};

constexpr int kSortWarps = 8;                                  // warps per block in the sort kernels
#ifndef TA_SORT_KEYS_PER_WARP
#define TA_SORT_KEYS_PER_WARP 384   // 256: 111.6 us, 384: 106.3 us, 512: 115.9 us per c3 sort (round 2)
#endif
constexpr int kSortKeysPerWarp = TA_SORT_KEYS_PER_WARP;                          // depth sort: keys per warp
constexpr int kSortKeysPerBlock = kSortWarps * kSortKeysPerWarp;   // keys per block (= partition)

// Number of LSD passes of 8 bits covering the varying bits of the visible depth keys.
__device__ __forceinline__ int sort_passes(const CallState* cs) {
    const uint32_t m = cs->key_or ^ cs->key_and;
    if (cs->n_visible == 0 || m == 0) return 0;
    const int lo = __ffs(m) - 1, hi = 31 - __clz(m);
    return (hi - lo) / 8 + 1;
}
__device__ __forceinline__ int sort_shift(const CallState* cs, int pass) {
    const uint32_t m = cs->key_or ^ cs->key_and;
    return (__ffs(m) - 1) + 8 * pass;
}

}  // namespace ta
