// composite.cu -- a6 front-to-back compositing of the C-channel latent feature (sm_100a), and the
// tile split that feeds it.
//
//   k_tile_split<NQ>   coarse (bin, depth, id) lists -> per-tile lists (tile q of bin b at
//                      NQ * start_b + q * len_b), trng[tile] = (start, count)
//   k_tile_order       heaviest-first order of the tiles (by list length)
//   k_composite_tc<C>  fp16-stored features: persistent warps, each pulling 8x8 pixel blocks (tile
//                      quadrants) from a per-call counter; lane l owns pixels (l&7, l>>3) and
//                      (l&7, (l>>3)+4).  The warp walks its tile's list, stages the entries whose
//                      ellipse can reach its still-active pixels (splat record + fp16 feature row by
//                      cp.async), runs the normative fp32 recurrence with packed fp32x2 instructions
//                      (T, alpha', the decisions and A bit-exact) and accumulates F on the tensor
//                      cores (mma.sync m16n8k16, fp16 hi/lo weights x fp16 features, fp32 accumulate;
//                      for C = 32 / 64 the accumulators live in tensor memory between chunks,
//                      tcgen05.ld / st, which frees the registers for a fifth CTA per SM).
//   k_composite<C, float>  fp32-stored features: the same recurrence, all-SIMT packed FFMA2
//                      accumulation, one CTA per tile.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "common.cuh"
#include "internal.h"
#include "tc_dev.cuh"

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

constexpr int kWarps = 4;                        // warps per CTA = 8x8-pixel blocks of the 16x16 tile
constexpr int kThreads = 32 * kWarps;
constexpr int kBuf = 64;                         // entries staged per warp at a time

template <int C>
struct WarpBuf {
    static constexpr int CP = C + 4;   // padded fp32 feature row
    float4 g[kBuf];                    // mx, my, ca, cb2
    float2 g2[kBuf];                   // cc, alpha
    uint2 bm[kBuf];                    // lanes whose pixel A / pixel B lies inside the pixel box
    float f[kBuf][CP];
};

// One CTA per 16x16 tile, warp w owning the 8x8 block (8*(w&1), 8*(w>>1)) -- or, for 8x8 tiles, one
// tile per warp (4 per CTA); lane l owns the two pixels
// (l&7, l>>3) and (l&7, (l>>3)+4) of its block (same column: dx is shared, the rest is computed
// for both pixels with packed fp32x2 instructions).  Warps are fully independent (no barrier):
// each walks the tile's (tile, depth, id) list (k_tile_split), keeps the entries whose ellipse can
// reach its still-active pixels (conservative), stages them in a warp-private shared buffer (splat
// record + fp32 feature row) and composites them; the 4 warps of a tile share the list reads
// through L1.
template <int C, typename FT, bool kCounts, bool kFast>
__global__ void __launch_bounds__(kThreads, (C >= 64 ? 2 : 4))
k_composite(const uint4* __restrict__ rec, const FT* __restrict__ feat, const uint32_t* __restrict__ clist,
            const uint2* __restrict__ trng, const uint32_t* __restrict__ order, CompositeGeom cg, RasterConsts rc,
            const CallState* __restrict__ cs, uint64_t list_cap, float* __restrict__ Fout, float* __restrict__ Aout,
            int32_t* __restrict__ ncontrib) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    WarpBuf<C>& bf = reinterpret_cast<WarpBuf<C>*>(smem_raw)[warp];

    // 16 x 16 tiles: one CTA per tile, warp w = quadrant w; 8 x 8 tiles: one tile per warp
    const bool t8 = cg.ts == 3;
    const uint32_t slot = t8 ? 4u * blockIdx.x + warp : blockIdx.x;
    if (slot >= (uint32_t)(cg.TX * cg.TY)) return;     // (warp-level: the kernel has no CTA barrier)
    const int tile = (int)order[slot];                 // heaviest tiles first (k_tile_order)
    const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
    const uint2 tr = trng[tile];                       // this tile's (depth, id)-ordered list (k_tile_split)
    const uint32_t cstart = tr.x;
    uint32_t cend = tr.x + tr.y;
    if (cend > list_cap) cend = (uint32_t)list_cap;   // overflowed async call: never read past the list
    const uint32_t n = cs->n;
    const int W = cg.W, H = cg.H;

    const int bx0 = (txi << cg.ts) + (t8 ? 0 : 8 * (int)(warp & 1)), by0 = (tyi << cg.ts) + (t8 ? 0 : 8 * (int)(warp >> 1));
    const int px = bx0 + (int)(lane & 7), pyA = by0 + (int)(lane >> 3), pyB = pyA + 4;
    const float pxf = (float)px;
    const float2 py2 = make_float2((float)pyA, (float)pyB);
    const float qlim = rc.q_max * 1.015625f + 0.01f;
    const uint32_t lt = lanemask_lt();

    float2 FA[C / 2], FB[C / 2];
#pragma unroll
    for (int c = 0; c < C / 2; c++) { FA[c] = make_float2(0.0f, 0.0f); FB[c] = make_float2(0.0f, 0.0f); }
    float2 T = make_float2(1.0f, 1.0f);
    int ncA = 0, ncB = 0;
    bool doneA = (px >= W) || (pyA >= H);
    bool doneB = (px >= W) || (pyB >= H);

    unsigned long long wk[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // kCounts: work counters (lane 0)
    uint32_t pos = cstart;
    while (pos < cend && !__all_sync(0xffffffffu, doneA && doneB)) {
        // culling rectangle = bounding box of the pixels still compositing (shrinks as pixels stop;
        // entries that can only reach stopped pixels are never staged)
        const bool actA = !doneA, actB = !doneB;
        const int ax0 = __reduce_min_sync(0xffffffffu, (actA || actB) ? px : 0x7fffffff);
        const int ax1 = __reduce_max_sync(0xffffffffu, (actA || actB) ? px : -1);
        const int ay0 = __reduce_min_sync(0xffffffffu, actA ? pyA : (actB ? pyB : 0x7fffffff));
        const int ay1 = __reduce_max_sync(0xffffffffu, actB ? pyB : (actA ? pyA : -1));
        const float X0 = (float)ax0, X1 = (float)ax1, Y0 = (float)ay0, Y1 = (float)ay1;
        // ---- fill: up to kBuf entries of this warp, in list order; 64 list entries (two independent
        //      32-entry chunks) per round trip
        int cnt = 0;
        while (cnt < kBuf && pos < cend) {
            uint32_t idx[2];
            uint4 r0[2], r1[2];
            bool keep[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t e = pos + 32 * h + lane;
                idx[h] = e < cend ? clist[e] : 0xffffffffu;
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t i = idx[h] < n ? idx[h] : 0u;
                r0[h] = rec[2 * i];
                r1[h] = rec[2 * i + 1];
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int gx0 = (int)(r1[h].z & 0xffff), gx1 = (int)(r1[h].z >> 16);
                const int gy0 = (int)(r1[h].w & 0xffff), gy1 = (int)(r1[h].w >> 16);
                keep[h] = (idx[h] < n) & (gx0 <= gx1) & ((gx0 >> cg.ts) <= txi) & (txi <= (gx1 >> cg.ts)) &
                          ((gy0 >> cg.ts) <= tyi) & (tyi <= (gy1 >> cg.ts)) & (gx0 <= ax1) & (gx1 >= ax0) & (gy0 <= ay1) &
                          (gy1 >= ay0) &
                          ellipse_may_touch_bf(__uint_as_float(r0[h].x), __uint_as_float(r0[h].y), __uint_as_float(r0[h].z),
                                               __uint_as_float(r0[h].w), __uint_as_float(r1[h].x), X0, X1, Y0, Y1, qlim);
            }
            uint32_t adv = 0;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                if (cnt >= kBuf) break;                   // warp-uniform
                const uint32_t base = pos + 32 * h;
                if (base >= cend) break;
                bool kp = keep[h];
                uint32_t bal = __ballot_sync(0xffffffffu, kp);
                const int room = kBuf - cnt;
                const uint32_t rank = __popc(bal & lt);
                uint32_t step = min(32u, cend - base);
                if (__popc(bal) > room) {                 // buffer full: resume at the first entry not taken
                    const uint32_t cut = __ballot_sync(0xffffffffu, kp && rank == (uint32_t)room);
                    const int cl = __ffs(cut) - 1;
                    bal &= (1u << cl) - 1u;
                    step = (uint32_t)cl;
                    kp = kp && (int)lane < cl;
                }
                if (kp) {
                    const int d = cnt + (int)rank;
                    bf.g[d] = make_float4(__uint_as_float(r0[h].x), __uint_as_float(r0[h].y), __uint_as_float(r0[h].z),
                                          __uint_as_float(r0[h].w));
                    bf.g2[d] = make_float2(__uint_as_float(r1[h].x), __uint_as_float(r1[h].y));
                    const int gx0 = (int)(r1[h].z & 0xffff), gx1 = (int)(r1[h].z >> 16);
                    const int gy0 = (int)(r1[h].w & 0xffff), gy1 = (int)(r1[h].w >> 16);
                    uint32_t mA, mB;
                    box_lane_masks(gx0, gx1, gy0, gy1, bx0, by0, mA, mB);
                    bf.bm[d] = make_uint2(mA, mB);
                    FeatLoad<FT>::template row<C>(feat + (size_t)idx[h] * C, &bf.f[d][0]);
                }
                cnt += __popc(bal);
                adv += step;
                if (step < 32u) break;                     // partial chunk: the next round resumes here
            }
            pos += adv;
            if (kCounts) { wk[0] += adv; wk[7] += 1; }
        }
        if (kCounts) wk[1] += cnt;
        __syncwarp();
        // ---- composite the staged entries in order, two pixels per lane
#pragma unroll 2
        for (int j = 0; j < cnt; j++) {
            const float4 G = bf.g[j];
            const float2 G2 = bf.g2[j];
            const uint2 bm = bf.bm[j];
            bool inA = !doneA && ((bm.x >> lane) & 1u), inB = !doneB && ((bm.y >> lane) & 1u);
            // q = fma(fma(ca, dx, cb2*dy), dx, (cc*dy)*dy), both pixels
            const float dx = fsub(pxf, G.x);
            const float2 dy = sub2(py2, bc2(G.y));
            const float2 t1 = mul2(bc2(G.w), dy);
            const float2 t2 = fma2(bc2(G.z), bc2(dx), t1);
            const float2 t4 = mul2(mul2(bc2(G2.x), dy), dy);
            const float2 q = fma2(t2, bc2(dx), t4);
            inA = inA && q.x <= rc.q_max;
            inB = inB && q.y <= rc.q_max;
            if (kCounts) wk[2] += 1;
            if (!__any_sync(0xffffffffu, inA || inB)) continue;
            if (kCounts) wk[3] += 1;
            const float2 e = exp2v<kFast>(mul2(bc2(-0.5f), q));
            const float2 ae = mul2(bc2(G2.y), e);
            const float2 a = make_float2(fminf(rc.alpha_max, ae.x), fminf(rc.alpha_max, ae.y));
            inA = inA && a.x >= rc.alpha_min;
            inB = inB && a.y >= rc.alpha_min;
            const float2 Tn = mul2(T, sub2(bc2(1.0f), a));
            const bool stopA = inA && Tn.x < rc.t_eps, stopB = inB && Tn.y < rc.t_eps;
            doneA = doneA || stopA;
            doneB = doneB || stopB;
            inA = inA && !stopA;
            inB = inB && !stopB;
            const float2 w = mul2(a, T);
            const float wA = inA ? w.x : 0.0f, wB = inB ? w.y : 0.0f;   // weight 0: exact no-op FMA
            const bool anyA = __any_sync(0xffffffffu, inA), anyB = __any_sync(0xffffffffu, inB);
            const float4* fr = reinterpret_cast<const float4*>(&bf.f[j][0]);
            if (anyA && anyB) {
#pragma unroll
                for (int c = 0; c < C / 4; c++) {
                    const float4 f4 = fr[c];
                    const float2 lo = make_float2(f4.x, f4.y), hi = make_float2(f4.z, f4.w);
                    FA[2 * c] = ffma2(lo, wA, FA[2 * c]);
                    FA[2 * c + 1] = ffma2(hi, wA, FA[2 * c + 1]);
                    FB[2 * c] = ffma2(lo, wB, FB[2 * c]);
                    FB[2 * c + 1] = ffma2(hi, wB, FB[2 * c + 1]);
                }
            } else if (anyA) {
#pragma unroll
                for (int c = 0; c < C / 4; c++) {
                    const float4 f4 = fr[c];
                    FA[2 * c] = ffma2(make_float2(f4.x, f4.y), wA, FA[2 * c]);
                    FA[2 * c + 1] = ffma2(make_float2(f4.z, f4.w), wA, FA[2 * c + 1]);
                }
            } else if (anyB) {
#pragma unroll
                for (int c = 0; c < C / 4; c++) {
                    const float4 f4 = fr[c];
                    FB[2 * c] = ffma2(make_float2(f4.x, f4.y), wB, FB[2 * c]);
                    FB[2 * c + 1] = ffma2(make_float2(f4.z, f4.w), wB, FB[2 * c + 1]);
                }
            }
            T = make_float2(inA ? Tn.x : T.x, inB ? Tn.y : T.y);
            if (kCounts) {
                wk[4] += (anyA || anyB) ? 1 : 0;
                wk[5] += __popc(__ballot_sync(0xffffffffu, inA)) + __popc(__ballot_sync(0xffffffffu, inB));
                ncA += inA ? 1 : 0;
                ncB += inB ? 1 : 0;
            }
            if (__all_sync(0xffffffffu, doneA && doneB)) break;
        }
        __syncwarp();
    }

    if (kCounts && lane == 0) {
        unsigned long long* work = const_cast<CallState*>(cs)->work;
        wk[6] = 1;
#pragma unroll
        for (int k = 0; k < 8; k++) atomicAdd(&work[k], wk[k]);
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int py = h ? pyB : pyA;
        if (px < W && py < H) {
            const size_t pix = (size_t)py * W + px;
            float4* out = reinterpret_cast<float4*>(Fout + pix * C);
            const float2* Fp = h ? FB : FA;
#pragma unroll
            for (int c = 0; c < C / 4; c++) out[c] = make_float4(Fp[2 * c].x, Fp[2 * c].y, Fp[2 * c + 1].x, Fp[2 * c + 1].y);
            Aout[pix] = fsub(1.0f, h ? T.y : T.x);
            if (kCounts) ncontrib[pix] = h ? ncB : ncA;
        }
    }
}

// Per-tile lists from the coarse (2^shift-pixel) bin lists, in list order: the (tile, depth, id)
// order of SURVEY a3-a5 (an entry belongs to tile t iff its pixel box covers t).  One 1024-thread
// block per coarse bin; its list is cut into 32 contiguous segments, one per warp: pass 1 counts each
// segment's entries per tile (the NQ = 2^sb x 2^sb tiles of the bin, from the tile rectangle
// k_bin_place stored above the entry's index), an exclusive scan over the warps gives every (segment, tile) write
// offset, pass 2 writes.  Tile q of bin b owns tlist[NQ cstart_b + q len_b, + len_b) (a tile list
// is a subsequence of the bin list); trng[tile] = (start, count).
#ifndef TA_SPLIT_PACKED
#define TA_SPLIT_PACKED 1
#endif
template <int NQ>
__global__ void __launch_bounds__(1024) k_tile_split(const uint32_t* __restrict__ clist,
                                                     const uint32_t* __restrict__ coffs, CompositeGeom cg,
                                                     const CallState* __restrict__ cs, uint64_t clist_cap,
                                                     uint32_t* __restrict__ tlist, uint64_t tlist_cap,
                                                     uint2* __restrict__ trng) {
    constexpr int SB = NQ == 4 ? 1 : 2, TPB = 1 << SB, IB = entry_idx_bits(SB);
    __shared__ uint32_t s_cnt[32][NQ];
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int bin = blockIdx.x;
    const int bxi = bin % cg.BX, byi = bin / cg.BX;
    const uint32_t P = cs->bin_P;                     // bin-major [NB x P] run starts (this call's P)
    const uint32_t cstart = coffs[(size_t)bin * P];
    uint32_t cend = coffs[(size_t)(bin + 1) * P];
    if (cend > clist_cap) cend = (uint32_t)clist_cap;
    const uint32_t len = cend > cstart ? cend - cstart : 0u;
    const uint32_t segl = (((len + 31u) / 32u) + 31u) & ~31u;          // entries per warp (multiple of 32)
    const uint32_t s0 = cstart + warp * segl, s1 = min(cend, s0 + segl);
    const uint32_t lt = lanemask_lt();
    const uint64_t tbase = (uint64_t)cstart * NQ;
    // every write of this bin lies below tbase + NQ len: one capacity check for the whole bin
    const bool fits = tbase + (uint64_t)NQ * len <= tlist_cap && (uint64_t)NQ * len < (1ull << 32);
    uint32_t* const tl = tlist + (fits ? tbase : 0);
    constexpr int kU = 4;                                           // chunks of 32 entries in flight
    // pass 2 keeps in run[q] the offset of tile q's next entry from tl (q len + cursor)
    auto walk = [&](bool write, uint32_t (&run)[NQ]) {
        for (uint32_t pos = s0; pos < s1; pos += 32 * kU) {
            uint32_t ent[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const uint32_t e = pos + 32 * u + lane;
                ent[u] = e < s1 ? clist[e] : 0u;          // 0: no tiles (padding)
            }
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const uint32_t idx = ent[u] & ((1u << IB) - 1u), r = ent[u] >> IB;
                uint32_t tm = r;                                   // sb = 1: the tile mask
                if (SB == 2) {                                     // sb = 2: tile rectangle -> 16-bit mask
                    const uint32_t x0 = r & 3u, x1 = (r >> 2) & 3u, y0 = (r >> 4) & 3u, y1 = r >> 6;
                    const uint32_t mx = (2u << x1) - (1u << x0);
                    tm = 0u;
#pragma unroll
                    for (int qy = 0; qy < TPB; qy++)
                        if ((uint32_t)qy >= y0 && (uint32_t)qy <= y1) tm |= mx << (qy * TPB);
                    if (pos + 32 * u + lane >= s1) tm = 0u;
                }
                if (NQ == 16 && __all_sync(0xffffffffu, tm == (1u << NQ) - 1u)) {   // 32 entries covering the whole bin
#pragma unroll
                    for (int q = 0; q < NQ; q++) {
                        if (write && fits) tl[run[q] + lane] = idx;
                        run[q] += 32u;
                    }
                    continue;
                }
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const bool ok = (tm >> q) & 1u;
                    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                    if (write && ok && fits) tl[run[q] + __popc(bal & lt)] = idx;
                    run[q] += __popc(bal);
                }
            }
        }
    };
    uint32_t run[NQ];
#pragma unroll
    for (int q = 0; q < NQ; q++) run[q] = 0u;
    if (NQ == 4 && TA_SPLIT_PACKED) {
        // pass 1 for 2 x 2 tiles: each lane counts its entries per tile in two 16-bit-field words, one warp
        // reduction per tile at the end (instead of a ballot per tile per 32 entries)
        uint32_t c01 = 0u, c23 = 0u;
        for (uint32_t pos = s0 + lane; pos < s1; pos += 32) {
            const uint32_t tm = clist[pos] >> IB;
            c01 += (tm & 1u) | ((tm & 2u) << 15);
            c23 += ((tm >> 2) & 1u) | ((tm & 8u) << 13);
        }
        run[0] = __reduce_add_sync(0xffffffffu, c01 & 0xffffu);
        run[1] = __reduce_add_sync(0xffffffffu, c01 >> 16);
        run[2 % NQ] = __reduce_add_sync(0xffffffffu, c23 & 0xffffu);
        run[3 % NQ] = __reduce_add_sync(0xffffffffu, c23 >> 16);
    } else {
        walk(false, run);
    }
#pragma unroll
    for (int q = 0; q < NQ; q++)
        if (lane == (uint32_t)q) s_cnt[warp][q] = run[q];
    __syncthreads();
    if (warp == 0) {                                              // exclusive scan over the 32 segments, per tile
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            const uint32_t v = s_cnt[lane][q];
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            s_cnt[lane][q] = x - v;
            if (lane == 31) {
                const int tx = (bxi << SB) + (q & ((1 << SB) - 1)), ty = (byi << SB) + (q >> SB);
                if (tx < cg.TX && ty < cg.TY)
                    trng[ty * cg.TX + tx] = make_uint2((uint32_t)min(tbase + (uint64_t)q * len, (uint64_t)0xffffffffu), x);
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; q++) run[q] = (uint32_t)q * len + s_cnt[warp][q];
    walk(true, run);
}

// Launch order of the tile CTAs: by decreasing log2 of the tile's list length (longest
// lists first, so the last wave is made of short tiles).  One block; order within a bucket is
// arbitrary (it only affects scheduling, never results).
#ifndef TA_ORDER_CAP
#define TA_ORDER_CAP 2048
#endif
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ trng, CompositeGeom cg,
                                                     uint32_t* __restrict__ order) {
    __shared__ uint32_t s_cnt[33], s_off[33];
    const int T = cg.TX * cg.TY;
    if (threadIdx.x < 33) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    auto bucket = [&](int t) {
        // the list length saturates as a cost estimate: a fully covered block stops long before the end
        // of a long list (c3: 0.904 -> 0.895 ms with the cap at 2048 entries)
        const uint32_t len = min(trng[t].y, (uint32_t)TA_ORDER_CAP);
        return 32 - (32 - __clz(len));                 // 32 - bit length: longer lists -> smaller bucket
    };
    for (int t = threadIdx.x; t < T; t += blockDim.x) atomicAdd(&s_cnt[bucket(t)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 0; b < 33; b++) { s_off[b] = run; run += s_cnt[b]; }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += blockDim.x) order[atomicAdd(&s_off[bucket(t)], 1u)] = (uint32_t)t;
}

// ============================================================================ tensor-core variant
// k_composite_tc<C>: fp16-stored features.  The per-pixel recurrence (q, exp_det, alpha', T, the
// stop rule) is the same packed fp32 sequence as k_composite, so T and A stay bit-exact; only the
// C-channel accumulation F[pixel][c] += w[pixel][j] * f[j][c] moves to the tensor cores.  Per 16
// staged entries it is a dense contraction F[64 px x C] += W[64 px x 16] . f[16 x C], done with
// mma.sync m16n8k16 (fp16 x fp16 -> fp32).  The fp16 features are exact operands; the fp32 weight
// w is split into w_hi = fp16(2^11 w) and w_lo = fp16(2^11 w - w_hi), both multiplied by the same
// f (two MMAs), so each weight keeps ~22 significant bits; the 2^11 scale keeps w_lo clear of the
// fp16 subnormals and is removed exactly at the end.  Products are exact and the MMA accumulates
// in fp32, so F matches the oracle's sequential fp32 sum to ~1e-6 (tolerance 1e-4, R22).

#ifndef TA_TC_NB
#define TA_TC_NB 64
#endif
template <int N>
struct SAcc {
    float4 v[N][32];
};
template <>
struct SAcc<0> {};

template <int C, int NBO = 0, bool TM = false>
struct TcBuf {
    // fp16 feature row pitch (halves): an odd number of 16-B chunks, so the 8 rows one ldmatrix
    // phase reads fall into 8 different 16-B bank groups
    static constexpr int PH = (((C + 8) / 8) & 1) ? C + 8 : C + 16;
    static constexpr int WP = 36;      // weight row pitch (32-bit words): 144 B, odd number of 16-B chunks
    // C = 64: the accumulators of channels 32..63 live in shared memory (lane-private float4 slots)
    // and 32 entries are staged at a time, so 3 CTAs fit per SM instead of 2 (registers / smem)
#ifndef TA_TC_NTR32
#define TA_TC_NTR32 4
#endif
    // (TM: every accumulator in tensor memory, none in shared memory)
    static constexpr int NT = C / 8, NTR = TM ? NT : (C >= 64 ? 4 : (C == 32 ? TA_TC_NTR32 : NT)), NTS = NT - NTR;
    static constexpr int NB = NBO > 0 ? NBO : (C >= 64 ? 32 : TA_TC_NB);   // entries staged per warp at a time
    // staged records, entry pairs (2k, 2k+1) interleaved so that the compacted mode loads its packed
    // (entry, entry) operands directly: p[k][0] = (mx, mx', my, my'), [1] = (-ca/2, .., -cb2/2, ..),
    // [2] = (-cc/2, .., 2^11 alpha, ..), [3] = (box lane mask A, .., mask B, ..)  (pre-scaled by exact
    // powers of two: q' = -q/2, a' = 2^11 alpha')
    float4 p[NB / 2][4];
    __half f[NB][PH];                  // staged fp16 feature rows
    uint32_t w[2][16][WP];             // [hi|lo][k][lane]: half2 (w(pixel A), w(pixel B)) of staged entry j0+k
    SAcc<4 * NTS> sacc;                // [mt * NTS + nt - NTR][lane] (C = 64 only)
    unsigned long long mbar;           // TA_TC_STAGE 2: completion of the fill's bulk feature-row copies
};

// Feature-row staging of the fill: 0 = cp.async 16 B x (2C / 16) per entry, waited for before the
// first compositing chunk; 1 = the same, waited for just before the first chunk's MMA (the weights
// of that chunk are computed meanwhile); 2 = one bulk copy (cp.async.bulk, TMA) per entry completing
// on a per-warp mbarrier, waited for before the first chunk's MMA.
#ifndef TA_TC_STAGE
#define TA_TC_STAGE 0
#endif

// Skip the exp / recurrence of an entry pair no pixel can take (saves ~13 % of pairs, but the
// warp-wide vote + branch splits the unrolled loop into basic blocks the scheduler cannot overlap;
// round 2 also measured a q-based skip -- compute both entries' q first, skip when no active in-box
// pixel has q <= q_max: 1.005 -> 1.11 ms on c3 -- a per-row refinement of the fill's cull, the
// active x span of each block row tested at the clamped 1D minimiser: 1.005 -> 1.46 ms -- and a
// relevance pre-pass over each fill round's staged entries (q of every entry for the active pixels,
// the kept slots compacted into a permutation the branch-free recurrence walks): 1.005 -> 1.51 ms,
// the pre-pass alone costing ~29 warp instructions per staged entry).
constexpr bool kSkipEmptyPairs = false;
#ifndef TA_TC_MIN_BLOCKS
#define TA_TC_MIN_BLOCKS 4
#endif
constexpr int kTcMinBlocks = TA_TC_MIN_BLOCKS;   // CTAs per SM the register budget targets

// kTm (fp16 C = 32 and 64, the default there): the 64 x C fp32 accumulators of a warp's block live in
// tensor memory (the warp's lane quarter, 2C columns per CTA) instead of registers (C = 32: 64 of them)
// or registers + shared memory (C = 64); each 16-entry chunk loads one 16-pixel m-tile (C / 2 columns)
// at a time (tcgen05.ld), runs its mma.sync and stores it back (tcgen05.st).  C = 32: 96 registers and
// 32 staged entries (8 KB of shared memory) per warp, 5 CTAs (20 warps) per SM instead of 4 (c3:
// 1.013 -> 0.981 ms; 6 CTAs at 80 registers spill: 1.166 ms).  C = 64: 128 TMEM columns per CTA, so
// 4 CTAs per SM instead of 3.
#ifndef TA_TM_BLOCKS
#define TA_TM_BLOCKS 5
#endif
#ifndef TA_TM_NB
#define TA_TM_NB 32
#endif
constexpr int kTmBlocks = TA_TM_BLOCKS;
template <int C, bool kTm>
using TcBufT = TcBuf<C, kTm ? TA_TM_NB : 0, kTm>;
template <int C>
__host__ __device__ constexpr int tm_cols() { return C >= 64 ? 128 : 64; }    // TMEM columns per CTA (a power of two >= 32)

template <int C, bool kCounts, bool kFast, bool kTm>
__global__ void __launch_bounds__(kThreads, (kTm ? (C >= 64 ? 4 : kTmBlocks) : (C >= 64 ? 3 : kTcMinBlocks)))
k_composite_tc(const uint4* __restrict__ rec, const __half* __restrict__ feat, const uint32_t* __restrict__ clist,
               const uint2* __restrict__ trng, const uint32_t* __restrict__ order, CompositeGeom cg, RasterConsts rc,
               const CallState* __restrict__ cs, uint64_t list_cap, float* __restrict__ Fout, float* __restrict__ Aout,
               int32_t* __restrict__ ncontrib) {
    using Buf = TcBufT<C, kTm>;
    static_assert(!kTm || C == 32 || C == 64, "tensor-memory accumulators: C = 32 or 64");
    constexpr uint32_t kMtCols = C / 2;      // TMEM columns of one 16-pixel m-tile (NT n-tiles x 4 floats)
    constexpr int NT = C / 8;                 // n-tiles of 8 channels
    constexpr int PH = Buf::PH;
    constexpr int WP = Buf::WP;
    constexpr int NB = Buf::NB, NTR = Buf::NTR, NTS = Buf::NTS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    Buf& bf = reinterpret_cast<Buf*>(smem_raw)[warp];
    __shared__ uint32_t s_tmem;
    uint32_t tacc = 0;                        // kTm: this warp's accumulator columns (lane quarter warp & 3)
    if (kTm) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "n"(tm_cols<C>()) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tacc = s_tmem + ((32u * (warp & 3u)) << 16);
    }
    const uint32_t mbar = smem_u32(&bf.mbar);
    uint32_t mphase = 0u;
    if (TA_TC_STAGE == 2) {
        if (lane == 0) mbar_init1(mbar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }

    // Persistent warps: each warp takes the next 8 x 8 block (an 8 x 8 tile, or a quadrant of a 16 x 16
    // tile) in the heaviest-first tile order from a per-call counter until all are done, so a warp
    // that finishes early starts new work instead of idling until its CTA's slowest warp is done.
    uint32_t* const wq = &const_cast<CallState*>(cs)->scan_counter[6];
    const bool t8 = cg.ts == 3;
    const uint32_t nblk = (t8 ? 1u : 4u) * (uint32_t)(cg.TX * cg.TY);
    for (;;) {
        uint32_t blk = 0;
        if (lane == 0) blk = atomicAdd(wq, 1u);
        blk = __shfl_sync(0xffffffffu, blk, 0);
        if (blk >= nblk) break;
        const int tile = (int)order[t8 ? blk : blk >> 2];
        const uint32_t qd = t8 ? 0u : blk & 3u;            // the 8 x 8 quadrant of a 16 x 16 tile
        const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
        const uint2 tr = trng[tile];                       // this tile's (depth, id)-ordered list (k_tile_split)
        const uint32_t cstart = tr.x;
        uint32_t cend = tr.x + tr.y;
        if (cend > list_cap) cend = (uint32_t)list_cap;
        const uint32_t n = cs->n;
        const int W = cg.W, H = cg.H;

        const int bx0 = (txi << cg.ts) + 8 * (int)(qd & 1), by0 = (tyi << cg.ts) + 8 * (int)(qd >> 1);
        const int px = bx0 + (int)(lane & 7), pyA = by0 + (int)(lane >> 3), pyB = pyA + 4;
        const float pxf = (float)px;
        const float2 py2 = make_float2((float)pyA, (float)pyB);
        const float qmax = rc.q_max, teps = rc.t_eps;
        const float qlo = rc.q_lo_half, amx = rc.a_max_2k, alo = rc.a_min_2k;
        const float qlim = qmax * 1.015625f + 0.01f;
        const uint32_t lt = lanemask_lt();

        // ldmatrix row addresses.  A (weights, stored [k][pixel p' = 2 lane + (0: A, 1: B)]): lane i
        // addresses row k = (i & 7) + 8 (i >> 4) of matrix i >> 3, pixel chunk 2 mt + ((i >> 3) & 1).
        const int li = (int)lane;
        const uint32_t a_base = smem_u32(&bf.w[0][(li & 7) + 8 * (li >> 4)][0]) + (uint32_t)(((li >> 3) & 1) * 16);
        constexpr uint32_t kLoOff = 16 * WP * 4;
        // B (features, stored [k][channel]): lane i addresses row (i & 7) + 8 ((i >> 3) & 1), channel chunk 2 np + (i >> 4)
        const int bk = (li & 7) + 8 * ((li >> 3) & 1);
        const uint32_t b_base = smem_u32(&bf.f[0][0]) + (uint32_t)((li >> 4) * 16);
        uint32_t* const wst = &bf.w[0][0][li];    // this lane's word in weight row 0 (hi)

        float acc[kTm ? 1 : 4][NTR][4];
#pragma unroll
        for (int mt = 0; mt < (kTm ? 1 : 4); mt++)
#pragma unroll
            for (int nt = 0; nt < NTR; nt++)
#pragma unroll
                for (int e = 0; e < 4; e++) acc[mt][nt][e] = 0.0f;
        if constexpr (kTm) {
            float z[16];
#pragma unroll
            for (int i = 0; i < 16; i++) z[i] = 0.0f;
#pragma unroll
            for (int mt = 0; mt < 4; mt++)
#pragma unroll
                for (uint32_t c = 0; c < kMtCols; c += 16) tm_st16(tacc + kMtCols * mt + c, z);
        }
        if constexpr (NTS > 0) {
#pragma unroll
            for (int k = 0; k < 4 * NTS; k++) bf.sacc.v[k][li] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
        float2 T = make_float2(1.0f, 1.0f);
        int ncA = 0, ncB = 0;
        // active-pixel lane bits: the lane's bit while its pixel still composites, else 0
        uint32_t actA = (px < W && pyA < H) ? (1u << lane) : 0u;
        uint32_t actB = (px < W && pyB < H) ? (1u << lane) : 0u;

        // Compacted mode (entered once, when at most 32 of the 64 pixels still composite): each such pixel
        // moves to its own lane (original lane ol, half hs -> weight column p' = 2 ol + hs) and the packed
        // fp32x2 arithmetic runs over pairs of entries instead of pairs of pixels, so the warp walks the
        // rest of the list at twice the rate.  T and the decisions keep the same fp32 sequence.
        bool modeB = false, movedA = false, movedB = false, chas = false;
        int ol = 0, hs = 0, cpx = 0, cpy = 0, nc1 = 0;
        float T1 = 1.0f;
        uint32_t act1 = 0u;

        unsigned long long wk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t pos = cstart;
        uint32_t pf_pos = 0xffffffffu, pf[2] = {0u, 0u};     // prefetched list indices of entries pf_pos + [0, 64)
        while (pos < cend && __any_sync(0xffffffffu, (actA | actB | act1) != 0u)) {
            // culling rectangle = bounding box of the pixels still compositing
            int lx0, lx1, ly0, ly1;
            if (!modeB) {
                lx0 = (actA | actB) ? px : 0x7fffffff;
                lx1 = (actA | actB) ? px : -1;
                ly0 = actA ? pyA : (actB ? pyB : 0x7fffffff);
                ly1 = actB ? pyB : (actA ? pyA : -1);
            } else {
                lx0 = act1 ? cpx : 0x7fffffff;
                lx1 = act1 ? cpx : -1;
                ly0 = act1 ? cpy : 0x7fffffff;
                ly1 = act1 ? cpy : -1;
            }
            const int ax0 = __reduce_min_sync(0xffffffffu, lx0);
            const int ax1 = __reduce_max_sync(0xffffffffu, lx1);
            const int ay0 = __reduce_min_sync(0xffffffffu, ly0);
            const int ay1 = __reduce_max_sync(0xffffffffu, ly1);
            const float X0 = (float)ax0, X1 = (float)ax1, Y0 = (float)ay0, Y1 = (float)ay1;
            // ---- fill: up to NB entries of this warp, in list order; 64 list entries per round trip.
            //      The list indices of the next 64 entries are loaded one round ahead (pf_pos / pf).
            int cnt = 0;
            if (TA_TC_STAGE == 2) fence_async_smem();   // earlier generic reads of the rows before the bulk writes
            while (cnt < NB && pos < cend) {
                uint32_t idx[2];
                if (pf_pos == pos) {
                    idx[0] = pf[0];
                    idx[1] = pf[1];
                } else {
#pragma unroll
                    for (int hh = 0; hh < 2; hh++) {
                        const uint32_t e = pos + 32 * hh + lane;
                        idx[hh] = e < cend ? clist[e] : 0xffffffffu;
                    }
                }
                uint4 r0[2], r1[2];
                bool keep[2];
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const uint32_t i = idx[hh] < n ? idx[hh] : 0u;
                    r1[hh] = rec[2 * i + 1];
                    r0[hh] = rec[2 * i];
                }
                pf_pos = pos + 64;
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const uint32_t e = pf_pos + 32 * hh + lane;
                    pf[hh] = e < cend ? clist[e] : 0xffffffffu;
                }
                // The warp's block lies inside the tile, so "box overlaps the active rectangle" implies
                // "box covers the tile": the per-tile list filter is implied (lists hold visible Gaussians only).
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const int gx0 = (int)(r1[hh].z & 0xffff), gx1 = (int)(r1[hh].z >> 16);
                    const int gy0 = (int)(r1[hh].w & 0xffff), gy1 = (int)(r1[hh].w >> 16);
                    keep[hh] = (idx[hh] < n) & (gx0 <= ax1) & (gx1 >= ax0) & (gy0 <= ay1) & (gy1 >= ay0) &
                               ellipse_may_touch_bf(__uint_as_float(r0[hh].x), __uint_as_float(r0[hh].y),
                                                  __uint_as_float(r0[hh].z), __uint_as_float(r0[hh].w),
                                                  __uint_as_float(r1[hh].x), X0, X1, Y0, Y1, qlim);
                }
                uint32_t adv = 0;
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    if (cnt >= NB) break;
                    const uint32_t base = pos + 32 * hh;
                    if (base >= cend) break;
                    bool kp = keep[hh];
                    uint32_t bal = __ballot_sync(0xffffffffu, kp);
                    const int room = NB - cnt;
                    const uint32_t rank = __popc(bal & lt);
                    uint32_t step = min(32u, cend - base);
                    if (__popc(bal) > room) {
                        const uint32_t cut = __ballot_sync(0xffffffffu, kp && rank == (uint32_t)room);
                        const int cl = __ffs(cut) - 1;
                        bal &= (1u << cl) - 1u;
                        step = (uint32_t)cl;
                        kp = kp && (int)lane < cl;
                    }
                    if (TA_TC_STAGE == 2 && lane == 0 && bal) mbar_expect_tx(mbar, (uint32_t)__popc(bal) * (uint32_t)(2 * C));
                    if (kp) {
                        const int d = cnt + (int)rank;
                        const int gx0 = (int)(r1[hh].z & 0xffff), gx1 = (int)(r1[hh].z >> 16);
                        const int gy0 = (int)(r1[hh].w & 0xffff), gy1 = (int)(r1[hh].w >> 16);
                        float* const pp = reinterpret_cast<float*>(&bf.p[d >> 1][0]) + (d & 1);
                        pp[0] = __uint_as_float(r0[hh].x);
                        pp[2] = __uint_as_float(r0[hh].y);
                        pp[4] = -0.5f * __uint_as_float(r0[hh].z);
                        pp[6] = -0.5f * __uint_as_float(r0[hh].w);
                        pp[8] = -0.5f * __uint_as_float(r1[hh].x);
                        pp[10] = 2048.0f * __uint_as_float(r1[hh].y);
                        uint32_t mA, mB;
                        box_lane_masks(gx0, gx1, gy0, gy1, bx0, by0, mA, mB);
                        pp[12] = __uint_as_float(mA);
                        pp[14] = __uint_as_float(mB);
                        const char* src = reinterpret_cast<const char*>(feat + (size_t)idx[hh] * C);
                        const uint32_t dst = smem_u32(&bf.f[d][0]);
                        if (TA_TC_STAGE == 2) {
                            bulk_g2s(dst, src, (uint32_t)(2 * C), mbar);
                        } else {
#pragma unroll
                            for (int c = 0; c < C * 2; c += 16) cp_async16(dst + c, src + c);
                        }
                    }
                    cnt += __popc(bal);
                    adv += step;
                    if (step < 32u) break;
                }
                pos += adv;
                if (kCounts) { wk[0] += adv; wk[7] += 1; }
            }
            if (kCounts) wk[1] += cnt;
            if (TA_TC_STAGE == 0) cp_async_wait_all();
            if (TA_TC_STAGE == 2 && lane == 0) mbar_arrive1(mbar);
            bool feat_ready = TA_TC_STAGE == 0;
            __syncwarp();
            // ---- composite the staged entries, 16 at a time: SIMT weights -> smem -> tensor cores
            for (int j0 = 0; j0 < cnt; j0 += 16) {
                const int nk = min(16, cnt - j0);
                if (!modeB) {
                    const uint32_t mA = __ballot_sync(0xffffffffu, actA != 0u), mB = __ballot_sync(0xffffffffu, actB != 0u);
                    const int nA = __popc(mA), na = nA + __popc(mB);
                    if (na <= 32) {                           // enter the compacted mode (warp-uniform)
                        modeB = true;
                        movedA = actA != 0u;
                        movedB = actB != 0u;
                        const bool has = li < na;
                        int src = 0;
                        hs = 0;
                        if (has) {
                            if (li < nA) src = (int)__fns(mA, 0, li + 1);
                            else { src = (int)__fns(mB, 0, li - nA + 1); hs = 1; }
                        }
                        const float tA = __shfl_sync(0xffffffffu, T.x, src), tB = __shfl_sync(0xffffffffu, T.y, src);
                        const int cA = __shfl_sync(0xffffffffu, ncA, src), cB = __shfl_sync(0xffffffffu, ncB, src);
                        ol = src;
                        T1 = hs ? tB : tA;
                        nc1 = hs ? cB : cA;
                        act1 = has ? 1u : 0u;
                        chas = has;
                        cpx = bx0 + (ol & 7);
                        cpy = by0 + (ol >> 3) + 4 * hs;
                        actA = actB = 0u;
                        // weight columns of pixels that stopped earlier are never written again: zero them all
                        uint4* wz = reinterpret_cast<uint4*>(&bf.w[0][0][0]);
                        for (int k = li; k < 2 * 16 * WP / 4; k += 32) wz[k] = make_uint4(0u, 0u, 0u, 0u);
                        __syncwarp();
                    }
                }
                if (modeB) {
                    const float cpxf = (float)cpx, cpyf = (float)cpy;
                    __half* const wh = reinterpret_cast<__half*>(&bf.w[0][0][0]) + 2 * ol + hs;   // column p', row 0 (hi)
#pragma unroll 2
                    for (int jj = 0; jj < 16; jj += 2) {
                        float w0 = 0.0f, w1 = 0.0f;
                        if (jj < nk) {
                            const bool has1 = jj + 1 < nk;
                            const float4* const pr = bf.p[(j0 + jj) >> 1];   // entries j, j+1 side by side
                            const float4 P0 = pr[0], P1 = pr[1], P2 = pr[2], P3 = pr[3];
                            // q of entries j, j+1 for this lane's pixel (normative a6 sequence per component)
                            const float2 dx = sub2(bc2(cpxf), make_float2(P0.x, P0.y));
                            const float2 dy = sub2(bc2(cpyf), make_float2(P0.z, P0.w));
                            const float2 t1 = mul2(make_float2(P1.z, P1.w), dy);
                            const float2 t2 = fma2(make_float2(P1.x, P1.y), dx, t1);
                            const float2 t4 = mul2(mul2(make_float2(P2.x, P2.y), dy), dy);
                            const float2 q = fma2(t2, dx, t4);     // q' = -q/2 (staged conic is -conic/2)
                            const uint32_t b0 = __float_as_uint(hs ? P3.z : P3.x), b1 = __float_as_uint(hs ? P3.w : P3.y);
                            const float qm0 = (act1 && ((b0 >> ol) & 1u)) ? q.x : -kInf;
                            const float qm1 = (act1 && has1 && ((b1 >> ol) & 1u)) ? q.y : -kInf;
                            if (kCounts) wk[2] += has1 ? 2 : 1;
                            if (!kSkipEmptyPairs || __any_sync(0xffffffffu, fmaxf(qm0, qm1) >= qlo)) {
                                const float2 e = exp2v<kFast>(q);
                                const float2 ae = mul2(make_float2(P2.z, P2.w), e);             // 2^11 alpha e
                                const float2 a = make_float2(fminf(amx, ae.x), fminf(amx, ae.y)); // 2^11 alpha'
                                const float2 om = fma2(a, bc2(-1.0f / 2048.0f), bc2(1.0f));      // fl(1 - alpha')
                                {
                                    const float Tn = fmul(T1, om.x);
                                    const bool ok = qm0 >= qlo && a.x >= alo;
                                    const bool in = ok && Tn >= teps;
                                    if (ok && !in) act1 = 0u;
                                    w0 = in ? fmul(a.x, T1) : 0.0f;
                                    T1 = in ? Tn : T1;
                                    if (kCounts) nc1 += in ? 1 : 0;
                                }
                                {
                                    const float Tn = fmul(T1, om.y);
                                    const bool ok = act1 && qm1 >= qlo && a.y >= alo;
                                    const bool in = ok && Tn >= teps;
                                    if (ok && !in) act1 = 0u;
                                    w1 = in ? fmul(a.y, T1) : 0.0f;
                                    T1 = in ? Tn : T1;
                                    if (kCounts) nc1 += in ? 1 : 0;
                                }
                            }
                        }
                        const __half2 hi = __floats2half2_rn(w0, w1);
                        const float2 hf = __half22float2(hi);
                        const __half2 lo = __floats2half2_rn(fsub(w0, hf.x), fsub(w1, hf.y));
                        if (chas) {
                            wh[jj * 2 * WP] = __low2half(hi);
                            wh[(jj + 1) * 2 * WP] = __high2half(hi);
                            wh[(16 + jj) * 2 * WP] = __low2half(lo);
                            wh[(16 + jj + 1) * 2 * WP] = __high2half(lo);
                        }
                    }
                } else {
                    // full chunks (16 staged entries) take a branch-free copy of the pair loop, so the
                    // scheduler can overlap consecutive pairs; the last, partial chunk keeps the guards
                    auto pairs = [&](auto full) {
                        constexpr bool kFull = decltype(full)::value;
#pragma unroll
                        for (int jj = 0; jj < 16; jj += 2) {
                            float2 w0 = make_float2(0.0f, 0.0f), w1 = make_float2(0.0f, 0.0f);
                            if (kFull || jj < nk) {                          // warp-uniform
                                const float4* const pr = bf.p[(j0 + jj) >> 1];   // entries j, j+1 side by side
                                const float4 P0 = pr[0], P1 = pr[1], P2 = pr[2], P3 = pr[3];
                                const float4 G0 = make_float4(P0.x, P0.z, P1.x, P1.z), G1 = make_float4(P0.y, P0.w, P1.y, P1.w);
                                const float4 H0 = make_float4(P2.x, P2.z, P3.x, P3.z), H1 = make_float4(P2.y, P2.w, P3.y, P3.w);
                                // q' = -q/2 of both entries for both pixels; a pixel takes part while it is inside
                                // the entry's box (lane masks) and still compositing (actA / actB), and q' >= -q_max/2
                                const float2 q0 = quad_q(G0, H0.x, pxf, py2), q1 = quad_q(G1, H1.x, pxf, py2);
                                const uint32_t mA0 = __float_as_uint(H0.z), mB0 = __float_as_uint(H0.w);
                                const bool has1 = kFull || jj + 1 < nk;
                                const uint32_t mA1 = has1 ? __float_as_uint(H1.z) : 0u, mB1 = has1 ? __float_as_uint(H1.w) : 0u;
                                if (kCounts) wk[2] += has1 ? 2 : 1;
                                if (!kSkipEmptyPairs || __any_sync(0xffffffffu, ((mA0 | mA1) & actA) | ((mB0 | mB1) & actB))) {
                                    // exp / alpha' of both entries are independent of T: computed side by side
                                    const float2 x0 = exp2v<kFast>(q0);
                                    const float2 x1 = exp2v<kFast>(q1);
                                    const float2 ae0 = mul2(bc2(H0.y), x0), ae1 = mul2(bc2(H1.y), x1);   // 2^11 alpha e
                                    const float2 a0 = make_float2(fminf(amx, ae0.x), fminf(amx, ae0.y));
                                    const float2 a1 = make_float2(fminf(amx, ae1.x), fminf(amx, ae1.y));
                                    if (kCounts) {
                                        wk[3] += __any_sync(0xffffffffu, ((mA0 & actA) && q0.x >= qlo) || ((mB0 & actB) && q0.y >= qlo)) ? 1 : 0;
                                        wk[3] += __any_sync(0xffffffffu, ((mA1 & actA) && q1.x >= qlo) || ((mB1 & actB) && q1.y >= qlo)) ? 1 : 0;
                                    }
                                    w0 = tstep<kCounts>(q0, a0, mA0, mB0, qlo, alo, teps, T, actA, actB, ncA, ncB, wk);
                                    // entry 1 sees the active bits after entry 0 (pixels that just stopped drop out)
                                    w1 = tstep<kCounts>(q1, a1, mA1, mB1, qlo, alo, teps, T, actA, actB, ncA, ncB, wk);
                                }
                            }
                            // split into fp16 hi / lo and store rows jj, jj+1
                            const __half2 h0 = __floats2half2_rn(w0.x, w0.y), h1 = __floats2half2_rn(w1.x, w1.y);
                            const float2 r0 = sub2(w0, __half22float2(h0)), r1 = sub2(w1, __half22float2(h1));
                            const __half2 l0 = __floats2half2_rn(r0.x, r0.y), l1 = __floats2half2_rn(r1.x, r1.y);
                            wst[jj * WP] = *reinterpret_cast<const uint32_t*>(&h0);
                            wst[(jj + 1) * WP] = *reinterpret_cast<const uint32_t*>(&h1);
                            wst[16 * WP + jj * WP] = *reinterpret_cast<const uint32_t*>(&l0);
                            wst[16 * WP + (jj + 1) * WP] = *reinterpret_cast<const uint32_t*>(&l1);
                        }
                    };
                    if (nk == 16) pairs(std::integral_constant<bool, true>());
                    else pairs(std::integral_constant<bool, false>());
                }
                if (!feat_ready) {                   // staged feature rows: first needed by this chunk's MMA
                    if (TA_TC_STAGE == 2) { mbar_wait_parity(mbar, mphase); mphase ^= 1u; }
                    else cp_async_wait_all();
                    feat_ready = true;
                }
                __syncwarp();
                // B fragments: feature rows j0 .. j0+15 (rows past cnt carry weight 0: clamp to a staged row)
                uint32_t bfr[NT][2];
                {
                    const int row = min(j0 + bk, cnt - 1);
                    const uint32_t rb = b_base + (uint32_t)(row * PH * 2);
                    if constexpr (NT == 1) {
                        ldsm_x2_t(rb, bfr[0][0], bfr[0][1]);
                    } else {
#pragma unroll
                        for (int np = 0; np < NT / 2; np++)
                            ldsm_x4_t(rb + np * 32, bfr[2 * np][0], bfr[2 * np][1], bfr[2 * np + 1][0], bfr[2 * np + 1][1]);
                    }
                }
                if constexpr (kTm) tm_wait_st();        // the previous chunk's stores precede these loads
#pragma unroll
                for (int mt = 0; mt < 4; mt++) {
                    uint32_t ah[4], al[4];
                    ldsm_x4_t(a_base + mt * 32, ah[0], ah[1], ah[2], ah[3]);
                    ldsm_x4_t(a_base + mt * 32 + kLoOff, al[0], al[1], al[2], al[3]);
                    if constexpr (kTm) {                  // this m-tile's accumulators: tensor memory -> MMA -> back
                        float v[kMtCols];
#pragma unroll
                        for (uint32_t c = 0; c < kMtCols; c += 16)
                            tm_ld16(tacc + kMtCols * mt + c, *reinterpret_cast<float (*)[16]>(v + c));
                        float (&am)[NTR][4] = *reinterpret_cast<float (*)[NTR][4]>(v);
#pragma unroll
                        for (int nt = 0; nt < NTR; nt++) {
                            hmma16816(am[nt], ah, bfr[nt][0], bfr[nt][1]);
                            hmma16816(am[nt], al, bfr[nt][0], bfr[nt][1]);
                        }
#pragma unroll
                        for (uint32_t c = 0; c < kMtCols; c += 16)
                            tm_st16(tacc + kMtCols * mt + c, *reinterpret_cast<const float (*)[16]>(v + c));
                    } else {
#pragma unroll
                        for (int nt = 0; nt < NTR; nt++) {
                            hmma16816(acc[mt][nt], ah, bfr[nt][0], bfr[nt][1]);
                            hmma16816(acc[mt][nt], al, bfr[nt][0], bfr[nt][1]);
                        }
                    }
                    if constexpr (NTS > 0) {
#pragma unroll
                        for (int nt = NTR; nt < NT; nt++) {        // C = 64: accumulators in shared memory
                            float4& slot = bf.sacc.v[mt * NTS + nt - NTR][li];
                            const float4 v = slot;
                            float d[4] = {v.x, v.y, v.z, v.w};
                            hmma16816(d, ah, bfr[nt][0], bfr[nt][1]);
                            hmma16816(d, al, bfr[nt][0], bfr[nt][1]);
                            slot = make_float4(d[0], d[1], d[2], d[3]);
                        }
                    }
                }
                __syncwarp();
                if (!__any_sync(0xffffffffu, (actA | actB | act1) != 0u)) break;
            }
            if (!feat_ready) {                       // no chunk ran: consume this fill's copies / barrier phase
                if (TA_TC_STAGE == 2) { mbar_wait_parity(mbar, mphase); mphase ^= 1u; }
                else cp_async_wait_all();
            }
            __syncwarp();
        }

        if (kCounts && lane == 0) {
            unsigned long long* work = const_cast<CallState*>(cs)->work;
            wk[6] = 1;
#pragma unroll
            for (int k = 0; k < 8; k++) atomicAdd(&work[k], wk[k]);
        }
        // accumulator (mt, row r in 0..15) <-> pixel p' = 16 mt + r = 2 l' + h: lane l' = 8 mt + (r >> 1), pixel A/B = r & 1
        const int g = li >> 2, t = li & 3;
        if constexpr (kTm) tm_wait_st();
#pragma unroll
        for (int mt = 0; mt < 4; mt++) {
            float tv[kTm ? kMtCols : 1];
            if constexpr (kTm) {
#pragma unroll
                for (uint32_t c = 0; c < kMtCols; c += 16)
                    tm_ld16(tacc + kMtCols * mt + c, *reinterpret_cast<float (*)[16]>(tv + c));
            }
            float (&acm)[NTR][4] = kTm ? *reinterpret_cast<float (*)[NTR][4]>(tv) : acc[kTm ? 0 : mt];
#pragma unroll
            for (int half = 0; half < 2; half++) {
                const int r = g + 8 * half;
                const int l2 = 8 * mt + (r >> 1);
                const int ox = bx0 + (l2 & 7), oy = by0 + (l2 >> 3) + 4 * (r & 1);
                if (ox < W && oy < H) {
                    float* out = Fout + ((size_t)oy * W + ox) * C + 2 * t;
#pragma unroll
                    for (int nt = 0; nt < NTR; nt++)
                        *reinterpret_cast<float2*>(out + 8 * nt) =
                            make_float2(acm[nt][2 * half] * (1.0f / 2048.0f), acm[nt][2 * half + 1] * (1.0f / 2048.0f));
                    if constexpr (NTS > 0) {
#pragma unroll
                        for (int nt = NTR; nt < NT; nt++) {
                            const float4 v = bf.sacc.v[mt * NTS + nt - NTR][li];
                            *reinterpret_cast<float2*>(out + 8 * nt) =
                                make_float2((half ? v.z : v.x) * (1.0f / 2048.0f), (half ? v.w : v.y) * (1.0f / 2048.0f));
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            const int py = hh ? pyB : pyA;
            if (px < W && py < H && !(hh ? movedB : movedA)) {        // moved pixels are written by their new lane
                const size_t pix = (size_t)py * W + px;
                Aout[pix] = fsub(1.0f, hh ? T.y : T.x);
                if (kCounts) ncontrib[pix] = hh ? ncB : ncA;
            }
        }
        if (modeB && chas) {
            const size_t pix = (size_t)cpy * W + cpx;
            Aout[pix] = fsub(1.0f, T1);
            if (kCounts) ncontrib[pix] = nc1;
        }

    }
    if (kTm) {                                 // every warp of the CTA is done with its columns
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(tm_cols<C>()) : "memory");
    }
}

template <int C, bool kTm>
static cudaError_t launch_tc(int tiles, int resident, bool fast, const uint4* rec, const void* feat, const uint32_t* list,
                             const uint2* offs, uint32_t* order, CompositeGeom cg, RasterConsts rc, const CallState* cs,
                             uint64_t list_cap, float* F, float* A, int32_t* ncontrib, cudaStream_t st) {
    const size_t smem = sizeof(TcBufT<C, kTm>) * kWarps;
    if (tiles == 0) return cudaSuccess;
    // persistent warps: as many CTAs as are co-resident (more would only find the block counter spent)
    const int grid = std::min(tiles, resident);
    k_tile_order<<<1, 1024, 0, st>>>(offs, cg, order);
    const __half* fh = static_cast<const __half*>(feat);
#define TA_TC(K, FA) k_composite_tc<C, K, FA, kTm><<<grid, kThreads, smem, st>>>(rec, fh, list, offs, order, cg, rc, cs, list_cap, F, A, ncontrib)
    if (ncontrib) {
        if (fast) TA_TC(true, true); else TA_TC(true, false);
    } else {
        if (fast) TA_TC(false, true); else TA_TC(false, false);
    }
#undef TA_TC
    return cudaGetLastError();
}

template <int C, typename FT>
static cudaError_t launch_one(int tiles, bool fast, const uint4* rec, const void* feat, const uint32_t* list,
                              const uint2* offs, uint32_t* order, CompositeGeom cg, RasterConsts rc,
                              const CallState* cs, uint64_t list_cap, float* F, float* A, int32_t* ncontrib,
                              cudaStream_t st) {
    const size_t smem = sizeof(WarpBuf<C>) * kWarps;
    if (tiles == 0) return cudaSuccess;
    k_tile_order<<<1, 1024, 0, st>>>(offs, cg, order);
    const FT* ff = static_cast<const FT*>(feat);
    const int grid = cg.ts == 3 ? (tiles + kWarps - 1) / kWarps : tiles;
#define TA_ONE(K, FA) k_composite<C, FT, K, FA><<<grid, kThreads, smem, st>>>(rec, ff, list, offs, order, cg, rc, cs, list_cap, F, A, ncontrib)
    if (ncontrib) {
        if (fast) TA_ONE(true, true); else TA_ONE(true, false);
    } else {
        if (fast) TA_ONE(false, true); else TA_ONE(false, false);
    }
#undef TA_ONE
    return cudaGetLastError();
}

// Per-device launch preparation (called by ta_context_create with the context's device current):
// the dynamic shared-memory opt-in of every compositor instantiation (cudaFuncSetAttribute acts on
// the current device only) and the co-resident CTA count of the persistent tensor-core compositor
// for each C, capped at ctas_per_sm_cap (> 0) per SM.
template <int C>
static cudaError_t prepare_one(int num_sms, int cap, int* resident) {
    const int smem_tc = (int)(sizeof(TcBuf<C>) * kWarps), smem = (int)(sizeof(WarpBuf<C>) * kWarps);
    const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_composite_tc<C, false, false, false>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, true, false, false>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, false, true, false>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, true, true, false>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite<C, float, false, false>, A, smem)) ||
        (e = cudaFuncSetAttribute(k_composite<C, float, true, false>, A, smem)) ||
        (e = cudaFuncSetAttribute(k_composite<C, float, false, true>, A, smem)) ||
        (e = cudaFuncSetAttribute(k_composite<C, float, true, true>, A, smem)))
        return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_composite_tc<C, false, false, false>, kThreads, smem_tc))) return e;
    if (cap > 0) per_sm = std::min(per_sm, cap);
    *resident = std::max(1, num_sms * std::max(1, per_sm));
    return cudaSuccess;
}

// The tensor-memory-accumulator instantiations (C = 32): co-resident CTAs from the kernel's registers and
// shared memory and the SM's TMEM columns (64 per CTA); the occupancy API reports 1 CTA / SM for kernels
// that allocate tensor memory.
template <int C>
static cudaError_t prepare_tc_tm(int num_sms, int cap, int* resident) {
    const int smem_tc = (int)(sizeof(TcBufT<C, true>) * kWarps);
    const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_composite_tc<C, false, false, true>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, true, false, true>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, false, true, true>, A, smem_tc)) ||
        (e = cudaFuncSetAttribute(k_composite_tc<C, true, true, true>, A, smem_tc)))
        return e;
    cudaFuncAttributes fa{};
    if ((e = cudaFuncGetAttributes(&fa, k_composite_tc<C, false, false, true>))) return e;
    int dev = 0, regs_sm = 0, smem_sm = 0, thr_sm = 0, blk_sm = 0, smem_rsv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    cudaDeviceGetAttribute(&blk_sm, cudaDevAttrMaxBlocksPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int regs_blk = ((fa.numRegs * 32 + 255) / 256 * 256) * kWarps;   // 256-register warp granules
    int per_sm = std::min(thr_sm / kThreads, blk_sm);
    per_sm = std::min(per_sm, regs_sm / std::max(1, regs_blk));
    per_sm = std::min(per_sm, smem_sm / (smem_tc + (int)fa.sharedSizeBytes + smem_rsv));
    per_sm = std::min(per_sm, 512 / tm_cols<C>());
    if (getenv("TA_DEBUG_PREP"))
        fprintf(stderr, "k_composite_tc<%d, tmem>: %d regs, %d B local, smem %d, %d CTAs/SM\n", C, fa.numRegs,
                (int)fa.localSizeBytes, smem_tc, per_sm);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    *resident = std::max(1, num_sms * std::max(1, per_sm));
    return cudaSuccess;
}

cudaError_t prepare_composite(int num_sms, int ctas_per_sm_cap, int resident[6]) {
    cudaError_t e;
    if ((e = prepare_one<8>(num_sms, ctas_per_sm_cap, &resident[0])) ||
        (e = prepare_one<16>(num_sms, ctas_per_sm_cap, &resident[1])) ||
        (e = prepare_one<32>(num_sms, ctas_per_sm_cap, &resident[2])) ||
        (e = prepare_one<64>(num_sms, ctas_per_sm_cap, &resident[3])) ||
        (e = prepare_tc_tm<32>(num_sms, ctas_per_sm_cap, &resident[4])) ||
        (e = prepare_tc_tm<64>(num_sms, ctas_per_sm_cap, &resident[5])))
        return e;
    return cudaSuccess;
}

void launch_tile_order(const uint2* trng, CompositeGeom cg, uint32_t* order, cudaStream_t st) {
    k_tile_order<<<1, 1024, 0, st>>>(trng, cg, order);
}

int c_slot(int C) { return C == 8 ? 0 : C == 16 ? 1 : C == 32 ? 2 : 3; }

cudaError_t launch_composite(int C, int fbytes, int tiles, const int* resident, bool fast, const uint4* rec,
                             const void* feat, const uint32_t* list, const uint2* offs, uint32_t* order, CompositeGeom cg,
                             RasterConsts rc, const CallState* cs, uint64_t list_cap, float* F, float* A,
                             int32_t* ncontrib, cudaStream_t st, bool tm_acc) {
    if (tm_acc && C == 32 && fbytes == 2)
        return launch_tc<32, true>(tiles, resident[4], fast, rec, feat, list, offs, order, cg, rc, cs, list_cap, F, A,
                                   ncontrib, st);
    if (tm_acc && C == 64 && fbytes == 2)
        return launch_tc<64, true>(tiles, resident[5], fast, rec, feat, list, offs, order, cg, rc, cs, list_cap, F, A,
                                   ncontrib, st);
#define TA_CASE(CC)                                                                                              \
    case CC:                                                                                                     \
        return fbytes == 2 ? launch_tc<CC, false>(tiles, resident[c_slot(CC)], fast, rec, feat, list, offs, order, cg, rc, cs, \
                                           list_cap, F, A, ncontrib, st)                                         \
                           : launch_one<CC, float>(tiles, fast, rec, feat, list, offs, order, cg, rc, cs, list_cap, F, A, \
                                                   ncontrib, st);
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

// Debug / test only: compact the per-tile lists the compositor walks (k_tile_split output) into one
// array: pass 0 writes the counts (then scanned into offsets), pass 1 copies.  One warp per tile.
__global__ void __launch_bounds__(256) k_debug_tile_lists(const uint2* __restrict__ trng, const uint32_t* __restrict__ tlist,
                                                          CompositeGeom cg, uint32_t* __restrict__ tile_offs,
                                                          uint32_t* __restrict__ out, uint64_t out_cap, int pass) {
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const int T = cg.TX * cg.TY;
    const int t = blockIdx.x * 8 + (int)warp;
    if (blockIdx.x == 0 && threadIdx.x == 0 && pass == 0) tile_offs[T] = 0u;
    if (t >= T) return;
    const uint2 tr = trng[t];
    if (pass == 0) {
        if (lane == 0) tile_offs[t] = tr.y;
        return;
    }
    const uint32_t o = tile_offs[t];
    for (uint32_t k = lane; k < tr.y; k += 32)
        if ((uint64_t)o + k < out_cap) out[o + k] = tlist[(size_t)tr.x + k];
}

void launch_debug_tile_lists(const uint2* trng, const uint32_t* tlist, CompositeGeom cg, uint32_t* tile_offs,
                             unsigned long long* status, uint32_t* counter, unsigned long long* total, uint32_t* out_list,
                             uint64_t out_cap, int pass, cudaStream_t st) {
    const int T = cg.TX * cg.TY;
    const int blocks = (T + 7) / 8;
    if (pass == 0) {
        k_debug_tile_lists<<<blocks, 256, 0, st>>>(trng, tlist, cg, tile_offs, out_list, out_cap, 0);
        launch_scan(tile_offs, nullptr, (uint32_t)T + 1, status, counter, total, st);
    } else {
        k_debug_tile_lists<<<blocks, 256, 0, st>>>(trng, tlist, cg, tile_offs, out_list, out_cap, 1);
    }
}

void launch_tile_split(const uint32_t* clist, const uint32_t* coffs, CompositeGeom cg,
                       const CallState* cs, uint64_t clist_cap, uint32_t* tlist, uint64_t tlist_cap, uint2* trng,
                       cudaStream_t st) {
    const int sb = cg.shift - cg.ts;
    const int NB = cg.BX * ((cg.TY + (1 << sb) - 1) >> sb);
    if (sb == 1)
        k_tile_split<4><<<NB, 1024, 0, st>>>(clist, coffs, cg, cs, clist_cap, tlist, tlist_cap, trng);
    else
        k_tile_split<16><<<NB, 1024, 0, st>>>(clist, coffs, cg, cs, clist_cap, tlist, tlist_cap, trng);
}

}  // namespace ta
