// composite.cu -- a6 front-to-back compositing of the C-channel latent feature (sm_100a).
//
// One CTA per 16x16 tile, one pixel per thread; warp w owns the 8x4 pixel block
// (8*(w&1), 4*(w>>1)) of the tile.
// The tile's (depth, id)-ordered list is consumed in batches of kBatch Gaussians staged in
// shared memory (splat record + feature row converted once to fp32, padded rows so the
// 128-bit staging stores are conflict-free).  While staging, every entry gets two 8-bit warp
// masks: "may touch" (pixel box overlaps the warp's block AND a conservative minimum of q over
// the block is <= 9) and "block inside the pixel box" (per-pixel box test skipped); each warp
// then walks only its entries (ballot + ffs).  Accumulation uses packed FFMA2 (fma.rn.f32x2).  Transmittance T,
// the decisions (box, q <= 9, alpha' >= 1/255, T*(1-alpha') < 1e-4) and A = 1 - T follow the
// normative fp32 sequence (DESIGN.md a6) bit for bit; the C accumulators are fp32 FMAs.
// Warps retire when all their pixels stopped (__all_sync); the CTA leaves the list as soon
// as every pixel stopped (__syncthreads_count).
#include "common.cuh"
#include "internal.h"

namespace ta {


template <typename FT>
struct FeatLoad;

template <>
struct FeatLoad<float> {
    // row of C floats -> s_row (fp32), 16 B at a time
    template <int C>
    __device__ __forceinline__ static void row(const float* __restrict__ src, float* __restrict__ dst) {
#pragma unroll
        for (int c = 0; c < C; c += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + c));
            *reinterpret_cast<float4*>(dst + c) = v;
        }
    }
};

template <>
struct FeatLoad<__half> {
    template <int C>
    __device__ __forceinline__ static void row(const __half* __restrict__ src, float* __restrict__ dst) {
#pragma unroll
        for (int c = 0; c < C; c += 8) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + c));
            const __half2* h = reinterpret_cast<const __half2*>(&v);
            const float2 a = __half22float2(h[0]), b = __half22float2(h[1]);
            const float2 d = __half22float2(h[2]), e = __half22float2(h[3]);
            *reinterpret_cast<float4*>(dst + c) = make_float4(a.x, a.y, b.x, b.y);
            *reinterpret_cast<float4*>(dst + c + 4) = make_float4(d.x, d.y, e.x, e.y);
        }
    }
};

// Packed fp32x2 FMA (sm_100a FFMA2): acc.xy += f.xy * w.
__device__ __forceinline__ float2 ffma2(float2 f, float w, float2 acc) {
    unsigned long long r;
    const unsigned long long fa = *reinterpret_cast<const unsigned long long*>(&f);
    const unsigned long long ac = *reinterpret_cast<const unsigned long long*>(&acc);
    const float2 ww = make_float2(w, w);
    const unsigned long long wb = *reinterpret_cast<const unsigned long long*>(&ww);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(fa), "l"(wb), "l"(ac));
    return *reinterpret_cast<float2*>(&r);
}

// Conservative cull of a Gaussian against an 8x4 pixel rectangle [X0,X1]x[Y0,Y1]: returns false
// only if every pixel of the rectangle is provably outside q <= q_max (with a 1.6% + 0.01 margin
// covering fp32 rounding of the per-pixel q); nearly degenerate conics
// (condition > 4096) are never culled here (the per-pixel test decides).
__device__ __forceinline__ bool ellipse_may_touch(float mx, float my, float ca, float cb2, float cc, float X0,
                                                  float X1, float Y0, float Y1, float qlim) {
    const float lx = X0 - mx, hx = X1 - mx, ly = Y0 - my, hy = Y1 - my;
    if (lx <= 0.0f && hx >= 0.0f && ly <= 0.0f && hy >= 0.0f) return true;
    const float cb = 0.5f * cb2;
    const float detc = ca * cc - cb * cb;
    if (!(detc * 4096.0f > ca * cc)) return true;
    // minimum of q on each edge (the other coordinate clamped to the edge's extent)
    const float ica = __frcp_rn(ca), icc = __frcp_rn(cc);
    float best = 3.0e38f;
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const float dx = e ? hx : lx;          // vertical edges x = const
        const float dy = fminf(fmaxf(-cb * dx * icc, ly), hy);
        best = fminf(best, dx * (ca * dx + cb2 * dy) + cc * dy * dy);
        const float ey = e ? hy : ly;          // horizontal edges y = const
        const float ex = fminf(fmaxf(-cb * ey * ica, lx), hx);
        best = fminf(best, ex * (ca * ex + cb2 * ey) + cc * ey * ey);
    }
    return best <= qlim;
}

// ------------------------------------------------------------------ mbarrier helpers (sm_90+)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}

constexpr int kSlots = 6;          // ring depth
constexpr int kSlotCoarse = 64;    // coarse-list entries scanned per slot (2 chunks of 32)
constexpr int kSlotEntries = 64;   // capacity: Gaussians staged per slot
constexpr int kConsumers = 8;      // consumer warps = 8x4-pixel blocks of the 16x16 tile
constexpr int kProducers = 2;      // producer warps (slot k is filled by warp k % kProducers)
constexpr int kCompositeThreads = 32 * (kConsumers + kProducers);

template <int C>
struct CompositeSmem {
    static constexpr int CP = C + 4;   // padded fp32 feature row
    float4 g[kSlots][kSlotEntries];    // mx, my, ca, cb2
    float2 g2[kSlots][kSlotEntries];   // cc, alpha
    uint2 rect[kSlots][kSlotEntries];  // x0|x1<<16, y0|y1<<16
    float f[kSlots][kSlotEntries][CP];
    uint64_t full[kSlots], empty[kSlots];
    int cnt[kSlots];                   // entries staged in the slot
    int ndone;                         // consumer warps whose 32 pixels all stopped
};

// Warp-specialised compositing.  Producer warps walk the tile's coarse (32x32-bin) list in
// depth order, 64 entries per slot, keep the Gaussians whose tile box covers this tile (the
// tile's (tile, depth, id) list) and whose ellipse can reach the tile (conservative), and stage
// their splat records + fp32 feature rows.  Consumer warps (8x4 pixels each) consume slots in
// order without waiting on each other.  Every slot is produced and consumed (empty once all
// pixels stopped), so no party can wait on a slot that never comes.
template <int C, typename FT>
__global__ void __launch_bounds__(kCompositeThreads, (C >= 64 ? 1 : 2))
k_composite(const uint4* __restrict__ rec, const FT* __restrict__ feat, const uint32_t* __restrict__ clist,
            const uint32_t* __restrict__ coffs, CompositeGeom cg, RasterConsts rc, const CallState* __restrict__ cs,
            uint64_t list_cap, float* __restrict__ Fout, float* __restrict__ Aout, int32_t* __restrict__ ncontrib) {
    using Smem = CompositeSmem<C>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const int tile = blockIdx.x;
    const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    // coarse bin of this tile and its (depth, id)-ordered Gaussian list
    const int sb = cg.shift - 4;
    const int bin = (tyi >> sb) * cg.BX + (txi >> sb);
    const uint32_t cstart = coffs[(size_t)bin * cg.P];
    uint32_t cend = coffs[(size_t)(bin + 1) * cg.P];
    if (cend > list_cap) cend = (uint32_t)list_cap;   // overflowed async call: never read past the list
    if (cend < cstart) cend = cstart;
    const int nslots = (int)((cend - cstart + kSlotCoarse - 1) / kSlotCoarse);
    const uint32_t n = cs->n;
    const int W = cg.W, H = cg.H;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kConsumers);
        }
        sm.ndone = 0;
    }
    __syncthreads();

    if (warp >= kConsumers) {
        // ------------------------------------------------------------ producers
        const uint32_t pw = warp - kConsumers;
        const uint32_t lt = lanemask_lt();
        const float TX0 = (float)(txi * kTile), TX1 = TX0 + 15.0f, TY0 = (float)(tyi * kTile), TY1 = TY0 + 15.0f;
        const float qlim = rc.q_max * 1.015625f + 0.01f;
        for (int k = (int)pw; k < nslots; k += kProducers) {
            const int s = k % kSlots;
            if (k >= kSlots) mbar_wait(&sm.empty[s], ((k / kSlots) - 1) & 1);
            int cnt = 0;
            if (*(volatile int*)&sm.ndone < kConsumers) {
                const uint32_t pos = cstart + (uint32_t)k * kSlotCoarse;
                uint32_t idx[2];
                uint4 r0[2], r1[2];
                bool pass[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t e = pos + 32 * h + lane;
                    idx[h] = e < cend ? clist[e] : 0xffffffffu;
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    pass[h] = idx[h] < n;                     // (>= n only after an overflow / past the end)
                    const uint32_t i = pass[h] ? idx[h] : 0u;
                    r0[h] = rec[2 * i];
                    r1[h] = rec[2 * i + 1];
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int x0 = (int)(r1[h].z & 0xffff), x1 = (int)(r1[h].z >> 16);
                    const int y0 = (int)(r1[h].w & 0xffff), y1 = (int)(r1[h].w >> 16);
                    pass[h] = pass[h] && x0 <= x1 && (x0 >> 4) <= txi && txi <= (x1 >> 4) && (y0 >> 4) <= tyi &&
                              tyi <= (y1 >> 4) &&
                              ellipse_may_touch(__uint_as_float(r0[h].x), __uint_as_float(r0[h].y),
                                                __uint_as_float(r0[h].z), __uint_as_float(r0[h].w),
                                                __uint_as_float(r1[h].x), TX0, TX1, TY0, TY1, qlim);
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t bal = __ballot_sync(0xffffffffu, pass[h]);
                    if (pass[h]) {
                        const int d = cnt + (int)__popc(bal & lt);
                        sm.g[s][d] = make_float4(__uint_as_float(r0[h].x), __uint_as_float(r0[h].y),
                                                 __uint_as_float(r0[h].z), __uint_as_float(r0[h].w));
                        sm.g2[s][d] = make_float2(__uint_as_float(r1[h].x), __uint_as_float(r1[h].y));
                        sm.rect[s][d] = make_uint2(r1[h].z, r1[h].w);
                        FeatLoad<FT>::template row<C>(feat + (size_t)idx[h] * C, &sm.f[s][d][0]);
                    }
                    cnt += __popc(bal);
                }
            }
            if (lane == 0) sm.cnt[s] = cnt;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[s]);
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // warp w owns the 8x4 pixel block (8*(w&1), 4*(w>>1)) of the tile
    const int bx0 = txi * kTile + 8 * (int)(warp & 1), by0 = tyi * kTile + 4 * (int)(warp >> 1);
    const int px = bx0 + (int)(lane & 7), py = by0 + (int)(lane >> 3);
    const float pxf = (float)px, pyf = (float)py;
    const float qlim = rc.q_max * 1.015625f + 0.01f;
    const float X0 = (float)bx0, X1 = (float)(bx0 + 7), Y0 = (float)by0, Y1 = (float)(by0 + 3);

    float2 F[C / 2];
#pragma unroll
    for (int c = 0; c < C / 2; c++) F[c] = make_float2(0.0f, 0.0f);
    float T = 1.0f;
    int nc = 0;
    bool done = (px >= W) || (py >= H);
    bool warp_done = __all_sync(0xffffffffu, done);
    if (warp_done && lane == 0) atomicAdd(&sm.ndone, 1);

    for (int k = 0; k < nslots; k++) {
        const int s = k % kSlots;
        mbar_wait(&sm.full[s], (k / kSlots) & 1);
        const int ne = sm.cnt[s];
        for (int g0 = 0; g0 < ne && !warp_done; g0 += 32) {
            // lanes over entries: cull against this warp's block
            bool keep = false, inbox = false;
            const int jl = g0 + (int)lane;
            if (jl < ne) {
                const float4 G = sm.g[s][jl];
                const float cc = sm.g2[s][jl].x;
                const uint2 rr = sm.rect[s][jl];
                const int gx0 = (int)(rr.x & 0xffff), gx1 = (int)(rr.x >> 16);
                const int gy0 = (int)(rr.y & 0xffff), gy1 = (int)(rr.y >> 16);
                keep = gx0 <= bx0 + 7 && gx1 >= bx0 && gy0 <= by0 + 3 && gy1 >= by0 &&
                       ellipse_may_touch(G.x, G.y, G.z, G.w, cc, X0, X1, Y0, Y1, qlim);
                inbox = gx0 <= bx0 && gx1 >= bx0 + 7 && gy0 <= by0 && gy1 >= by0 + 3;
            }
            uint32_t bits = __ballot_sync(0xffffffffu, keep);
            const uint32_t inbits = __ballot_sync(0xffffffffu, inbox);
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                const int j = g0 + b;
                const float4 G = sm.g[s][j];
                const float2 G2 = sm.g2[s][j];
                if (!done) {
                    bool inside = true;
                    if (!((inbits >> b) & 1u)) {
                        const uint2 rr = sm.rect[s][j];
                        inside = px >= (int)(rr.x & 0xffff) && px <= (int)(rr.x >> 16) &&
                                 py >= (int)(rr.y & 0xffff) && py <= (int)(rr.y >> 16);
                    }
                    if (inside) {
                        const float dx = fsub(pxf, G.x), dy = fsub(pyf, G.y);
                        const float q = ffma(ffma(G.z, dx, fmul(G.w, dy)), dx, fmul(fmul(G2.x, dy), dy));
                        if (q <= rc.q_max) {
                            const float e = exp_det(fmul(-0.5f, q));
                            const float a = fminf(rc.alpha_max, fmul(G2.y, e));
                            if (a >= rc.alpha_min) {
                                const float Tn = fmul(T, fsub(1.0f, a));
                                if (Tn < rc.t_eps) {
                                    done = true;
                                } else {
                                    const float w = fmul(a, T);
                                    const float4* fr = reinterpret_cast<const float4*>(&sm.f[s][j][0]);
#pragma unroll
                                    for (int c = 0; c < C / 4; c++) {
                                        const float4 f4 = fr[c];
                                        F[2 * c] = ffma2(make_float2(f4.x, f4.y), w, F[2 * c]);
                                        F[2 * c + 1] = ffma2(make_float2(f4.z, f4.w), w, F[2 * c + 1]);
                                    }
                                    T = Tn;
                                    nc++;
                                }
                            }
                        }
                    }
                }
                if (__all_sync(0xffffffffu, done)) {
                    warp_done = true;
                    if (lane == 0) atomicAdd(&sm.ndone, 1);
                    break;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }

    if (px < W && py < H) {
        const size_t pix = (size_t)py * W + px;
        float4* out = reinterpret_cast<float4*>(Fout + pix * C);
#pragma unroll
        for (int c = 0; c < C / 4; c++) out[c] = make_float4(F[2 * c].x, F[2 * c].y, F[2 * c + 1].x, F[2 * c + 1].y);
        Aout[pix] = fsub(1.0f, T);
        if (ncontrib) ncontrib[pix] = nc;
    }
}

template <int C, typename FT>
static cudaError_t launch_one(int tiles, const uint4* rec, const void* feat, const uint32_t* list,
                              const uint32_t* offs, CompositeGeom cg, RasterConsts rc, const CallState* cs,
                              uint64_t list_cap, float* F, float* A, int32_t* ncontrib, cudaStream_t st) {
    const size_t smem = sizeof(CompositeSmem<C>);
    static bool attr_set = false;   // per template instance; set once per process
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_composite<C, FT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (tiles == 0) return cudaSuccess;
    k_composite<C, FT><<<tiles, kCompositeThreads, smem, st>>>(rec, static_cast<const FT*>(feat), list, offs, cg,
                                                                   rc, cs, list_cap, F, A, ncontrib);
    return cudaGetLastError();
}

cudaError_t launch_composite(int C, int fbytes, int tiles, const uint4* rec, const void* feat,
                             const uint32_t* list, const uint32_t* offs, CompositeGeom cg, RasterConsts rc,
                             const CallState* cs, uint64_t list_cap, float* F, float* A, int32_t* ncontrib,
                             cudaStream_t st) {
#define TA_CASE(CC)                                                                                           \
    case CC:                                                                                                  \
        return fbytes == 2 ? launch_one<CC, __half>(tiles, rec, feat, list, offs, cg, rc, cs, list_cap, F, A, ncontrib, st) \
                           : launch_one<CC, float>(tiles, rec, feat, list, offs, cg, rc, cs, list_cap, F, A, ncontrib, st);
    switch (C) {
        TA_CASE(8)
        TA_CASE(16)
        TA_CASE(32)
        TA_CASE(64)
        default:
            return cudaErrorInvalidValue;
    }
#undef TA_CASE
}

}  // namespace ta

namespace ta {

// Debug / test only: materialise the per-tile lists exactly as the compositor's producer walks them
// (coarse bin list filtered by tile box; without the conservative ellipse prefilter), pass 0 counts,
// pass 1 writes.  One warp per tile.
__global__ void __launch_bounds__(256) k_debug_tile_lists(const uint4* __restrict__ rec, const uint32_t* __restrict__ clist,
                                                          const uint32_t* __restrict__ coffs, CompositeGeom cg,
                                                          const CallState* __restrict__ cs, uint32_t* __restrict__ tile_offs,
                                                          uint32_t* __restrict__ out, uint64_t out_cap, int pass) {
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int T = cg.TX * cg.TY;
    const int t = blockIdx.x * 8 + (int)warp;
    if (blockIdx.x == 0 && threadIdx.x == 0 && pass == 0) tile_offs[T] = 0u;
    if (t >= T) return;
    const int tyi = t / cg.TX, txi = t - tyi * cg.TX;
    const int sb = cg.shift - 4;
    const int bin = (tyi >> sb) * cg.BX + (txi >> sb);
    const uint32_t cstart = coffs[(size_t)bin * cg.P], cend = coffs[(size_t)(bin + 1) * cg.P];
    const uint32_t n = cs->n;
    const uint32_t lt = lanemask_lt();
    uint32_t run = pass ? tile_offs[t] : 0u;
    for (uint32_t pos = cstart; pos < cend; pos += 32) {
        const uint32_t e = pos + lane;
        bool ok = false;
        uint32_t i = 0;
        if (e < cend) {
            i = clist[e];
            if (i < n) {
                const uint4 r1 = rec[2 * i + 1];
                const int x0 = (int)(r1.z & 0xffff), x1 = (int)(r1.z >> 16);
                const int y0 = (int)(r1.w & 0xffff), y1 = (int)(r1.w >> 16);
                ok = x0 <= x1 && (x0 >> 4) <= txi && txi <= (x1 >> 4) && (y0 >> 4) <= tyi && tyi <= (y1 >> 4);
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        if (pass && ok) {
            const uint64_t p = (uint64_t)run + __popc(bal & lt);
            if (p < out_cap) out[p] = i;
        }
        run += __popc(bal);
    }
    if (pass == 0 && lane == 0) tile_offs[t] = run;
}

void launch_debug_tile_lists(const uint4* rec, const uint32_t* clist, const uint32_t* coffs, CompositeGeom cg,
                             const CallState* cs, uint32_t* tile_offs, unsigned long long* status, uint32_t* counter,
                             unsigned long long* total, uint32_t* out_list, uint64_t out_cap, int pass,
                             cudaStream_t st) {
    const int T = cg.TX * cg.TY;
    const int blocks = (T + 7) / 8;
    if (pass == 0) {
        k_debug_tile_lists<<<blocks, 256, 0, st>>>(rec, clist, coffs, cg, cs, tile_offs, out_list, out_cap, 0);
        launch_scan(tile_offs, nullptr, (uint32_t)T + 1, status, counter, total, st);
    } else {
        k_debug_tile_lists<<<blocks, 256, 0, st>>>(rec, clist, coffs, cg, cs, tile_offs, out_list, out_cap, 1);
    }
}

}  // namespace ta
