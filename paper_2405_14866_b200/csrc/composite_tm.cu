// composite_tm.cu -- a6 front-to-back compositing with the C-channel accumulators in tensor memory
// (sm_100a: tcgen05.mma, TMEM, mbarrier).
//
// k_composite_tm<C, kCounts, kFastExp>: fp16-stored features, C in {16, 32, 64}.
//   * One CTA (4 warps) per 16 x 16 tile at a time, persistent: CTAs pull tiles in heaviest-first order
//     from a per-call counter.  Warp w owns the 8 x 8 quadrant w; lane l the two pixels (l&7, l>>3) and
//     (l&7, (l>>3)+4) of it (same column: dx is shared, the rest is computed for both pixels with packed
//     fp32x2 instructions).
//   * The tile's (depth, id)-ordered list (k_tile_split) is read ONCE per CTA: 128 threads test 128
//     entries per step against the active-pixel rectangle of every quadrant (pixel box + conservative
//     ellipse test), and the kept entries are staged in shared memory -- the splat record, per-quadrant
//     lane masks and relevance bits, and the fp16 feature row (cp.async 16-byte chunks) written straight
//     into the canonical no-swizzle MN-major layout the tensor core reads as the B operand.
//   * Per 16 staged entries every warp runs the normative fp32 recurrence for its pixels (q, exp_det,
//     alpha', T, the stop rule -- the sequence of DESIGN.md, so T, A and every decision are those of the
//     oracle) and writes its pixels' weights 2^11 alpha' T as fp16 hi / lo rows of the A operand
//     (canonical no-swizzle K-major, one 16-byte store per 8 entries).  The LAST warp to finish the
//     chunk issues, from one thread, F[128 px x C] += W[128 x 16] . f[16 x C] for the pixel-A and
//     pixel-B halves of the tile (hi and lo: 4 x tcgen05.mma.cta_group::1.kind::f16, M = 128, N = C,
//     K = 16, fp32 accumulate in TMEM) and commits them to an mbarrier; a warp waits for that commit only
//     before it overwrites the weight rows with the next chunk.  The accumulators never occupy registers
//     (D row 32 w + l = pixel A / B of warp w, lane l: each warp reads back exactly its own TMEM lane
//     quarter with tcgen05.ld at the end of the tile).
//   * When at most 32 of a warp's 64 pixels still composite, the warp compacts them onto its lanes (one
//     pixel per lane) and the packed arithmetic runs over pairs of entries instead.
// fp16 features are exact operands, products are exact, accumulation is fp32: F agrees with the oracle's
// sequential fp32 sum to ~1e-6 (tolerance 1e-4, R22).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "common.cuh"
#include "internal.h"
#include "tc_dev.cuh"

namespace ta {
namespace tmc {

constexpr int kWarps = 4;
constexpr int kThreads = 128;
constexpr int kNB = 64;                        // entries staged per fill round

// ---------------------------------------------------------------- PTX wrappers (tcgen05, mbarrier)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity), "r"(100000u)           // suspend-time hint (ns): sleep until the phase completes
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "n"(NCOL) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOL>
__device__ __forceinline__ void tmem_free(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOL) : "memory");
}

// D[tmem] (+)= A[smem] . B[smem], kind::f16 (fp16 x fp16 -> fp32), issued by one thread.
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// Arrive on the mbarrier once every tcgen05.mma this thread issued before has completed.
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Shared-memory matrix descriptor, canonical layout without swizzle (version 1 = sm_100):
// start address, leading-dimension and stride-dimension byte offsets, all >> 4.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// Instruction descriptor kind::f16: D fp32 (bit 4), A = B = fp16, A K-major, B MN-major (bit 16),
// N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// 32 lanes x 32-bit, 16 / 32 consecutive columns of the warp's TMEM lane quarter -> registers
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- shared memory of one CTA
// Weight matrices (A operand), 4 x [128 rows x 16 k] fp16, canonical K-major without swizzle:
// element (row r, k) at (r >> 3) * 128 + (k >> 3) * 2048 + (r & 7) * 16 + (k & 7) * 2.
// Matrix 0 / 1 = hi / lo weights of the pixel-A rows, 2 / 3 = of the pixel-B rows; row 32 w + l =
// pixel A (B) of warp w, lane l.
constexpr uint32_t kWRowGroup = 128, kWKGroup = 2048, kWMat = 4096;

template <int C>
struct alignas(128) Smem {
    uint8_t w[4][kWMat];
    // Feature rows (B operand), per chunk of 16 staged entries a [k 16 x N = C] fp16 matrix, canonical
    // MN-major without swizzle: element (channel n, entry k) at (n >> 3) * 128 + (k >> 3) * (C / 8) * 128 +
    // (k & 7) * 16 + (n & 7) * 2.
    uint8_t f[kNB / 16][32 * C];
    // staged records, entry pairs (2k, 2k+1) side by side (pre-scaled by exact powers of two:
    // q' = -q/2, a' = 2^11 alpha'): p[k][0] = (mx, mx', my, my'), [1] = (-ca/2, .., -cb2/2, ..),
    // [2] = (-cc/2, .., 2^11 alpha, ..)
    float4 p[kNB / 2][3];
    // per quadrant q: (box lane mask of pixel-A rows, entry 2k | 2k+1, pixel-B rows, 2k | 2k+1)
    uint4 m[kNB / 2][kWarps];
    int rect[kWarps][4];                 // active-pixel rectangle of each quadrant (x0 > x1: none active)
    uint32_t wcnt[3][kWarps];            // [0] active pixels per warp; [1 + parity] kept entries per fill step
    uint2 pk[256];                       // re-packing: (pixel id | composited count << 8, T bits) of active pixels
    uint32_t cut, tile, arrive, tmem;
    unsigned long long mbar;
};

template <int C>
__host__ __device__ constexpr int tmem_cols() {
    return 2 * C <= 32 ? 32 : 2 * C <= 64 ? 64 : 2 * C <= 128 ? 128 : 256;
}

// One step of the normative recurrence for the lane's two pixels (staged scaling; see composite.cu
// tstep): returns the weights 2^11 alpha' T (0 where the pixel does not take this entry).
template <bool kCounts>
__device__ __forceinline__ float2 step2(float2 q, float2 a, uint32_t mA, uint32_t mB, float qlo, float alo, float teps,
                                        float2& T, uint32_t& actA, uint32_t& actB, int& ncA, int& ncB) {
    const float2 Tn = mul2(T, fma2(a, bc2(-1.0f / 2048.0f), bc2(1.0f)));
    const bool okA = (mA & actA) && q.x >= qlo && a.x >= alo, okB = (mB & actB) && q.y >= qlo && a.y >= alo;
    const bool inA = okA && Tn.x >= teps, inB = okB && Tn.y >= teps;
    if (okA && !inA) actA = 0u;           // T would drop below t_eps: stop before this Gaussian (R10)
    if (okB && !inB) actB = 0u;
    const float2 ws = mul2(a, T);
    const float2 w = make_float2(inA ? ws.x : 0.0f, inB ? ws.y : 0.0f);
    T = make_float2(inA ? Tn.x : T.x, inB ? Tn.y : T.y);
    if (kCounts) {
        ncA += inA ? 1 : 0;
        ncB += inB ? 1 : 0;
    }
    return w;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// fp16 hi / lo split of two weights of one pixel (entries j, j+1): hi = fp16(w), lo = fp16(w - hi)
__device__ __forceinline__ void split2(float w0, float w1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(w0, w1);
    const float2 hf = __half22float2(h);
    hi = h2u(h);
    lo = h2u(__floats2half2_rn(fsub(w0, hf.x), fsub(w1, hf.y)));
}

template <int C, bool kCounts, bool kFast>
__global__ void __launch_bounds__(kThreads, (C >= 64 ? 4 : 8))
k_composite_tm(const uint4* __restrict__ rec, const __half* __restrict__ feat, const uint32_t* __restrict__ tlist,
               const uint2* __restrict__ trng, const uint32_t* __restrict__ order, CompositeGeom cg, RasterConsts rc,
               const CallState* __restrict__ cs, uint64_t list_cap, float* __restrict__ Fout, float* __restrict__ Aout,
               int32_t* __restrict__ ncontrib) {
    constexpr int NCOL = tmem_cols<C>();
    constexpr uint32_t IDESC = idesc_f16(128, C);
    constexpr uint32_t kFKGroup = (C / 8) * 128;          // k-group stride of the feature chunk
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem<C>& s = *reinterpret_cast<Smem<C>*>(smem_raw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
    const uint32_t lt = lanemask_lt();
    const uint32_t bar = smem_u32(&s.mbar);

    if (tid == 0) {
        mbar_init(bar, 1);
        s.arrive = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc<NCOL>(smem_u32(&s.tmem));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;

    const uint32_t n = cs->n;
    const int W = cg.W, H = cg.H;
    const float qmax = rc.q_max, teps = rc.t_eps;
    const float qlo = rc.q_lo_half, amx = rc.a_max_2k, alo = rc.a_min_2k;
    const float qlim = qmax * 1.015625f + 0.01f;
    uint32_t* const wq = &const_cast<CallState*>(cs)->scan_counter[6];
    const uint32_t ntiles = (uint32_t)(cg.TX * cg.TY);
    uint32_t chunks = 0;                                  // MMA groups issued by this CTA so far (CTA-uniform)
    unsigned long long wk[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    for (;;) {
        if (tid == 0) s.tile = atomicAdd(wq, 1u);
        __syncthreads();
        const uint32_t blk = s.tile;
        if (blk >= ntiles) break;
        const int tile = (int)order[blk];
        const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
        const uint2 tr = trng[tile];
        const uint32_t cstart = tr.x;
        uint32_t cend = tr.x + tr.y;
        if (cend > list_cap) cend = (uint32_t)list_cap;
        const int tbx = txi * kTile, tby = tyi * kTile;

        // Pixel slots: each thread holds up to two of the tile's 256 pixels.  Pixel p = 64 q + 32 h + l is
        // (quadrant q, half h, lane l): x = tbx + 8 (q & 1) + (l & 7), y = tby + 8 (q >> 1) + (l >> 3) + 4 h;
        // its accumulator row is TMEM lane 32 q + l of D_h, its weights go to row 32 q + l of the hi / lo
        // matrices 2 h, 2 h + 1.  Initially thread (w, l) holds pixels (w, 0, l) and (w, 1, l); when fewer
        // warps suffice, the active pixels are re-packed two per thread onto the first warps.
        int sp0 = (int)(64 * warp + lane), sp1 = sp0 + 32;
        float2 T = make_float2(1.0f, 1.0f);
        int nc0 = 0, nc1 = 0;
        auto pix_x = [&](int p) { return tbx + 8 * ((p >> 6) & 1) + (p & 7); };
        auto pix_y = [&](int p) { return tby + 8 * (p >> 7) + ((p >> 3) & 3) + 4 * ((p >> 5) & 1); };
        bool act0 = pix_x(sp0) < W && pix_y(sp0) < H, act1 = pix_x(sp1) < W && pix_y(sp1) < H;
        uint32_t busy_warps = kWarps;                       // warps holding pixels (CTA-uniform)
        const uint32_t tile_chunk0 = chunks;

        uint32_t pos = cstart;
        for (;;) {                                         // fill rounds
            if (chunks > 0) mbar_wait(bar, (chunks - 1) & 1u);   // last MMA done: staging buffers free
            // ---- active pixels of the tile; re-pack them when fewer warps suffice
            const uint32_t b0 = __ballot_sync(0xffffffffu, act0), b1 = __ballot_sync(0xffffffffu, act1);
            const uint32_t wact = __popc(b0) + __popc(b1);
            int lx0 = 0x7fffffff, lx1 = -1, ly0 = 0x7fffffff, ly1 = -1;
            if (act0) { lx0 = min(lx0, pix_x(sp0)); lx1 = max(lx1, pix_x(sp0)); ly0 = min(ly0, pix_y(sp0)); ly1 = max(ly1, pix_y(sp0)); }
            if (act1) { lx0 = min(lx0, pix_x(sp1)); lx1 = max(lx1, pix_x(sp1)); ly0 = min(ly0, pix_y(sp1)); ly1 = max(ly1, pix_y(sp1)); }
            lx0 = __reduce_min_sync(0xffffffffu, lx0);
            lx1 = __reduce_max_sync(0xffffffffu, lx1);
            ly0 = __reduce_min_sync(0xffffffffu, ly0);
            ly1 = __reduce_max_sync(0xffffffffu, ly1);
            if (lane == 0) {
                s.rect[warp][0] = lx0; s.rect[warp][1] = lx1; s.rect[warp][2] = ly0; s.rect[warp][3] = ly1;
                s.wcnt[0][warp] = wact;
            }
            __syncthreads();
            uint32_t nact = 0, pre = 0;
            int rx0 = 0x7fffffff, rx1 = -1, ry0 = 0x7fffffff, ry1 = -1;
#pragma unroll
            for (int q = 0; q < kWarps; q++) {
                const uint32_t c = s.wcnt[0][q];
                pre += (q < (int)warp) ? c : 0u;
                nact += c;
                rx0 = min(rx0, s.rect[q][0]); rx1 = max(rx1, s.rect[q][1]);
                ry0 = min(ry0, s.rect[q][2]); ry1 = max(ry1, s.rect[q][3]);
            }
            if (nact == 0 || pos >= cend) break;           // tile done (CTA-uniform)
            const uint32_t need = (nact + 63u) >> 6;
            if (need < busy_warps) {
                // drop the stopped pixels (their A is final), compact the active ones two per thread
                if (!act0 && sp0 >= 0 && pix_x(sp0) < W && pix_y(sp0) < H) {
                    const size_t pix = (size_t)pix_y(sp0) * W + pix_x(sp0);
                    Aout[pix] = fsub(1.0f, T.x);
                    if (kCounts) ncontrib[pix] = nc0;
                }
                if (!act1 && sp1 >= 0 && pix_x(sp1) < W && pix_y(sp1) < H) {
                    const size_t pix = (size_t)pix_y(sp1) * W + pix_x(sp1);
                    Aout[pix] = fsub(1.0f, T.y);
                    if (kCounts) ncontrib[pix] = nc1;
                }
                const uint32_t r0 = pre + __popc(b0 & lt) + __popc(b1 & lt);
                if (act0) s.pk[r0] = make_uint2((uint32_t)sp0 | ((uint32_t)nc0 << 8), __float_as_uint(T.x));
                if (act1) s.pk[r0 + (act0 ? 1 : 0)] = make_uint2((uint32_t)sp1 | ((uint32_t)nc1 << 8), __float_as_uint(T.y));
                // rows of dropped pixels must read 0 from now on: clear every weight row (the last MMA is done)
                {
                    uint4* wz = reinterpret_cast<uint4*>(&s.w[0][0]);
#pragma unroll
                    for (int i = 0; i < (int)(4 * kWMat / 16 / kThreads); i++) wz[i * kThreads + tid] = make_uint4(0u, 0u, 0u, 0u);
                }
                __syncthreads();
                const uint32_t i0 = 2 * tid, i1 = 2 * tid + 1;
                sp0 = -1; sp1 = -1; act0 = act1 = false;
                if (i0 < nact) {
                    const uint2 v = s.pk[i0];
                    sp0 = (int)(v.x & 255u); nc0 = (int)(v.x >> 8); T.x = __uint_as_float(v.y); act0 = true;
                }
                if (i1 < nact) {
                    const uint2 v = s.pk[i1];
                    sp1 = (int)(v.x & 255u); nc1 = (int)(v.x >> 8); T.y = __uint_as_float(v.y); act1 = true;
                }
                busy_warps = need;
            }
            // per-slot constants: coordinates, mask word selector, weight-row offset
            const int q0 = sp0 >= 0 ? sp0 >> 6 : 0, q1 = sp1 >= 0 ? sp1 >> 6 : 0;
            const uint32_t hs0 = sp0 >= 0 ? (uint32_t)(sp0 >> 5) & 1u : 0u, hs1 = sp1 >= 0 ? (uint32_t)(sp1 >> 5) & 1u : 0u;
            const uint32_t ls0 = (uint32_t)sp0 & 31u, ls1 = (uint32_t)sp1 & 31u;
            const float2 px2 = make_float2((float)pix_x(sp0 >= 0 ? sp0 : 0), (float)pix_x(sp1 >= 0 ? sp1 : 0));
            const float2 py2 = make_float2((float)pix_y(sp0 >= 0 ? sp0 : 0), (float)pix_y(sp1 >= 0 ? sp1 : 0));
            const uint32_t row0 = 32u * (uint32_t)q0 + ls0, row1 = 32u * (uint32_t)q1 + ls1;
            const uint32_t off0 = 2u * hs0 * kWMat + (row0 >> 3) * kWRowGroup + (row0 & 7u) * 16u;
            const uint32_t off1 = 2u * hs1 * kWMat + (row1 >> 3) * kWRowGroup + (row1 & 7u) * 16u;

            long long tf0 = kCounts ? clock64() : 0;
            // ---- fill: up to kNB entries, 128 list entries per step, in list order; an entry is kept when its
            //      pixel box meets the tile's active rectangle and its ellipse may reach it (conservative)
            const float X0 = (float)rx0, X1 = (float)rx1, Y0 = (float)ry0, Y1 = (float)ry1;
            uint32_t cnt = 0, par = 0;
            uint32_t nidx = pos + tid < cend ? tlist[pos + tid] : 0xffffffffu;
            while (cnt < (uint32_t)kNB && pos < cend) {
                const uint32_t idx = nidx;
                const uint32_t nxt = pos + kThreads + tid;
                nidx = nxt < cend ? tlist[nxt] : 0xffffffffu;   // prefetch (a cut step re-reads)
                uint4 r0 = make_uint4(0u, 0u, 0u, 0u), r1 = make_uint4(0u, 0u, 0u, 0u);
                bool keep = false;
                if (idx < n) {
                    r1 = rec[2 * idx + 1];
                    r0 = rec[2 * idx];
                    const int gx0 = (int)(r1.z & 0xffff), gx1 = (int)(r1.z >> 16);
                    const int gy0 = (int)(r1.w & 0xffff), gy1 = (int)(r1.w >> 16);
                    keep = gx0 <= rx1 && gx1 >= rx0 && gy0 <= ry1 && gy1 >= ry0 &&
                           ellipse_may_touch2(__uint_as_float(r0.x), __uint_as_float(r0.y), __uint_as_float(r0.z),
                                              __uint_as_float(r0.w), __uint_as_float(r1.x), X0, X1, Y0, Y1, qlim);
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                if (lane == 0) s.wcnt[1 + par][warp] = __popc(bal);
                __syncthreads();
                uint32_t tot = 0, wpre = 0;
#pragma unroll
                for (int v = 0; v < kWarps; v++) {
                    const uint32_t c = s.wcnt[1 + par][v];
                    wpre += (v < (int)warp) ? c : 0u;
                    tot += c;
                }
                const uint32_t grank = wpre + __popc(bal & lt);
                const uint32_t room = (uint32_t)kNB - cnt;
                uint32_t step = min((uint32_t)kThreads, cend - pos);
                if (tot > room) {                          // buffer full: resume at the first entry not taken
                    if (keep && grank == room) s.cut = tid;
                    __syncthreads();
                    step = s.cut;
                    tot = room;
                    const uint32_t e2 = pos + step + tid;
                    nidx = e2 < cend ? tlist[e2] : 0xffffffffu;
                }
                if (keep && grank < room) {
                    const uint32_t d = cnt + grank, k = d >> 1, h = d & 1u;
                    float* const pp = reinterpret_cast<float*>(&s.p[k][0]) + h;
                    pp[0] = __uint_as_float(r0.x);
                    pp[2] = __uint_as_float(r0.y);
                    pp[4] = -0.5f * __uint_as_float(r0.z);
                    pp[6] = -0.5f * __uint_as_float(r0.w);
                    pp[8] = -0.5f * __uint_as_float(r1.x);
                    pp[10] = 2048.0f * __uint_as_float(r1.y);
                    const int gx0 = (int)(r1.z & 0xffff), gx1 = (int)(r1.z >> 16);
                    const int gy0 = (int)(r1.w & 0xffff), gy1 = (int)(r1.w >> 16);
#pragma unroll
                    for (int q = 0; q < kWarps; q++) {
                        uint32_t* const mm = reinterpret_cast<uint32_t*>(&s.m[k][q]);
                        const int qx = tbx + 8 * (q & 1), qy = tby + 8 * (q >> 1);
                        mm[h] = box_lane_mask(gx0, gx1, gy0, gy1, qx, qy);
                        mm[2 + h] = box_lane_mask(gx0, gx1, gy0, gy1, qx, qy + 4);
                    }
                    const char* src = reinterpret_cast<const char*>(feat + (size_t)idx * C);
                    const uint32_t fb = smem_u32(&s.f[d >> 4][0]) + ((d >> 3) & 1u) * kFKGroup + (d & 7u) * 16u;
#pragma unroll
                    for (int c = 0; c < C / 8; c++) cp_async16(fb + (uint32_t)c * 128u, src + 16 * c);
                }
                cnt += tot;
                pos += step;
                par ^= 1u;
                if (kCounts && tid == 0) { wk[0] += step; wk[7] += 1; }
            }
            if (kCounts && tid == 0) wk[1] += cnt;
            // entries cnt .. end of the last chunk: zero feature rows (they carry weight 0; no NaN x 0)
            {
                const uint32_t cend16 = (cnt + 15u) & ~15u;
                for (uint32_t d = cnt + (tid >> 3); d < cend16; d += kThreads / 8) {
                    const uint32_t c = tid & 7u;
                    if (c < (uint32_t)(C / 8))
                        *reinterpret_cast<uint4*>(&s.f[d >> 4][((d >> 3) & 1u) * kFKGroup + c * 128u + (d & 7u) * 16u]) =
                            make_uint4(0u, 0u, 0u, 0u);
                }
            }
            cp_async_wait_all();
            fence_proxy_async_smem();
            __syncthreads();
            if (kCounts && lane == 0) wk[2] += clock64() - tf0;

            // ---- composite the staged entries, 16 at a time
            const uint32_t nchunk = (cnt + 15u) >> 4;
            const bool busy = warp < busy_warps;
            long long tc0 = kCounts ? clock64() : 0;
            for (uint32_t j = 0; j < nchunk; j++) {
                const int j0 = (int)(16u * j);
                const int nk = min(16, (int)cnt - j0);
                if (busy) {
#pragma unroll
                    for (int b = 0; b < 2; b++) {
                        uint32_t hi[2][4], lo[2][4];       // [slot][entry pair]: fp16 (entry 2i, 2i+1)
#pragma unroll
                        for (int jp = 0; jp < 4; jp++) {
                            const int jj = 8 * b + 2 * jp;
                            float2 w0 = make_float2(0.0f, 0.0f), w1 = make_float2(0.0f, 0.0f);
                            const int k = (j0 + jj) >> 1;
                            if (jj < nk) {                 // warp-uniform
                                const uint4 M0 = s.m[k][q0], M1 = s.m[k][q1];
                                const bool has1 = jj + 1 < nk;
                                // box lane-mask bits of each slot's pixel for entries 2k, 2k+1
                                const uint32_t e00 = ((hs0 ? M0.z : M0.x) >> ls0) & 1u, e01 = ((hs0 ? M0.w : M0.y) >> ls0) & 1u;
                                const uint32_t e10 = ((hs1 ? M1.z : M1.x) >> ls1) & 1u, e11 = ((hs1 ? M1.w : M1.y) >> ls1) & 1u;
                                const uint32_t m0A = act0 ? e00 : 0u, m0B = act1 ? e10 : 0u;
                                const uint32_t m1A = (act0 && has1) ? e01 : 0u, m1B = (act1 && has1) ? e11 : 0u;
                                if (__any_sync(0xffffffffu, (m0A | m0B | m1A | m1B) != 0u)) {
                                    const float4 P0 = s.p[k][0], P1 = s.p[k][1], P2 = s.p[k][2];
                                    // q' = -q/2 of entries 2k (P*.x / .z) and 2k+1 (.y / .w) for both slots
                                    float2 q0v, q1v;
                                    {
                                        const float2 dx = sub2(px2, bc2(P0.x)), dy = sub2(py2, bc2(P0.z));
                                        const float2 t1 = mul2(bc2(P1.z), dy);
                                        const float2 t2 = fma2(bc2(P1.x), dx, t1);
                                        const float2 t4 = mul2(mul2(bc2(P2.x), dy), dy);
                                        q0v = fma2(t2, dx, t4);
                                    }
                                    {
                                        const float2 dx = sub2(px2, bc2(P0.y)), dy = sub2(py2, bc2(P0.w));
                                        const float2 t1 = mul2(bc2(P1.w), dy);
                                        const float2 t2 = fma2(bc2(P1.y), dx, t1);
                                        const float2 t4 = mul2(mul2(bc2(P2.y), dy), dy);
                                        q1v = fma2(t2, dx, t4);
                                    }
                                    const float2 x0 = exp2v<kFast>(q0v);
                                    const float2 x1 = exp2v<kFast>(q1v);
                                    const float2 ae0 = mul2(bc2(P2.z), x0), ae1 = mul2(bc2(P2.w), x1);
                                    const float2 a0 = make_float2(fminf(amx, ae0.x), fminf(amx, ae0.y));
                                    const float2 a1 = make_float2(fminf(amx, ae1.x), fminf(amx, ae1.y));
                                    uint32_t A0 = act0 ? 1u : 0u, A1 = act1 ? 1u : 0u;
                                    w0 = step2<kCounts>(q0v, a0, m0A, m0B, qlo, alo, teps, T, A0, A1, nc0, nc1);
                                    w1 = step2<kCounts>(q1v, a1, m1A, m1B, qlo, alo, teps, T, A0, A1, nc0, nc1);
                                    act0 = A0 != 0u;
                                    act1 = A1 != 0u;
                                }
                            }
                            split2(w0.x, w1.x, hi[0][jp], lo[0][jp]);
                            split2(w0.y, w1.y, hi[1][jp], lo[1][jp]);
                        }
                        long long tw0 = kCounts ? clock64() : 0;
                        if (b == 0 && chunks > 0) mbar_wait(bar, (chunks - 1) & 1u);   // rows free again
                        if (kCounts && lane == 0) wk[4] += clock64() - tw0;
                        if (sp0 >= 0) {
                            *reinterpret_cast<uint4*>(&s.w[0][off0 + (uint32_t)b * kWKGroup]) = make_uint4(hi[0][0], hi[0][1], hi[0][2], hi[0][3]);
                            *reinterpret_cast<uint4*>(&s.w[0][off0 + kWMat + (uint32_t)b * kWKGroup]) = make_uint4(lo[0][0], lo[0][1], lo[0][2], lo[0][3]);
                        }
                        if (sp1 >= 0) {
                            *reinterpret_cast<uint4*>(&s.w[0][off1 + (uint32_t)b * kWKGroup]) = make_uint4(hi[1][0], hi[1][1], hi[1][2], hi[1][3]);
                            *reinterpret_cast<uint4*>(&s.w[0][off1 + kWMat + (uint32_t)b * kWKGroup]) = make_uint4(lo[1][0], lo[1][1], lo[1][2], lo[1][3]);
                        }
                    }
                } else if (chunks > 0) {
                    long long tw0 = kCounts ? clock64() : 0;
                    mbar_wait(bar, (chunks - 1) & 1u);     // arrivals of chunk j only after chunk j-1's MMAs
                    if (kCounts && lane == 0) wk[5] += clock64() - tw0;
                }
                // ---- hand the chunk to the tensor core: the last warp to arrive issues the MMAs
                fence_proxy_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    const uint32_t old = atomicAdd(&s.arrive, 1u);
                    if ((old & 3u) == 3u) {
                        __threadfence_block();
                        tc_fence_after();
                        const uint32_t acc = chunks > tile_chunk0 ? 1u : 0u;
                        const uint64_t bd = sdesc(smem_u32(&s.f[j][0]), kFKGroup, 128u);
#pragma unroll
                        for (int hh = 0; hh < 2; hh++) {
                            const uint32_t dt = tmem + (uint32_t)(hh * C);
                            umma_f16(dt, sdesc(smem_u32(&s.w[2 * hh][0]), kWKGroup, kWRowGroup), bd, IDESC, acc);
                            umma_f16(dt, sdesc(smem_u32(&s.w[2 * hh + 1][0]), kWKGroup, kWRowGroup), bd, IDESC, 1u);
                        }
                        umma_commit(bar);
                    }
                }
                __syncwarp();
                chunks++;
            }
            if (kCounts && tid == 0) wk[6] += nchunk;
            if (kCounts && lane == 0) wk[3] += clock64() - tc0;
        }

        // ---- epilogue: F from this warp's TMEM lane quarter (pixels (warp, h, lane)), A of the held pixels
        if (chunks > tile_chunk0) {
            mbar_wait(bar, (chunks - 1) & 1u);
            tc_fence_after();
        }
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
            const int p = (int)(64 * warp + 32 * hh + lane);
            const int px = pix_x(p), py = pix_y(p);
            const bool inside = px < W && py < H;
            float* const out = Fout + ((size_t)py * W + px) * C;
#pragma unroll
            for (int c0 = 0; c0 < C; c0 += 16) {
                float v[16];
                if (chunks > tile_chunk0) {
                    tmem_ld16(tmem + ((32u * warp) << 16) + (uint32_t)(hh * C + c0), v);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; i++) v[i] = 0.0f;
                }
                if (inside) {
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4*>(out + c0 + i) =
                            make_float4(v[i] * (1.0f / 2048.0f), v[i + 1] * (1.0f / 2048.0f), v[i + 2] * (1.0f / 2048.0f),
                                        v[i + 3] * (1.0f / 2048.0f));
                }
            }
        }
        if (sp0 >= 0 && pix_x(sp0) < W && pix_y(sp0) < H) {
            const size_t pix = (size_t)pix_y(sp0) * W + pix_x(sp0);
            Aout[pix] = fsub(1.0f, T.x);
            if (kCounts) ncontrib[pix] = nc0;
        }
        if (sp1 >= 0 && pix_x(sp1) < W && pix_y(sp1) < H) {
            const size_t pix = (size_t)pix_y(sp1) * W + pix_x(sp1);
            Aout[pix] = fsub(1.0f, T.y);
            if (kCounts) ncontrib[pix] = nc1;
        }
        tc_fence_before();
        __syncthreads();                                   // TMEM reads done before the next tile's first MMA
    }

    if (kCounts && tid == 0) {                             // [0] list entries read, [1] staged, [6] MMA chunks,
        unsigned long long* work = const_cast<CallState*>(cs)->work;   // [7] fill steps (this kernel)
        atomicAdd(&work[0], wk[0]);
        atomicAdd(&work[1], wk[1]);
        atomicAdd(&work[6], wk[6]);
        atomicAdd(&work[7], wk[7]);
    }
    if (kCounts && lane == 0) {                            // cycles per warp: [2] fill, [3] composite rounds,
        unsigned long long* work = const_cast<CallState*>(cs)->work;   // [4] of which waiting before stores,
        atomicAdd(&work[2], wk[2]);                        // [5] of which idle-warp waits
        atomicAdd(&work[3], wk[3]);
        atomicAdd(&work[4], wk[4]);
        atomicAdd(&work[5], wk[5]);
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_free<NCOL>(tmem);
    }
}

}  // namespace tmc

template <int C>
static cudaError_t prepare_tm_one(int num_sms, int cap, int* resident) {
    const size_t smem = sizeof(tmc::Smem<C>) + 1024;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(tmc::k_composite_tm<C, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) ||
        (e = cudaFuncSetAttribute(tmc::k_composite_tm<C, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) ||
        (e = cudaFuncSetAttribute(tmc::k_composite_tm<C, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) ||
        (e = cudaFuncSetAttribute(tmc::k_composite_tm<C, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
        return e;
    // Co-resident CTAs per SM from the kernel's registers and shared memory and the SM's limits, and the
    // TMEM columns (512 per SM).  (cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 for kernels that
    // allocate tensor memory, which would leave 7/8 of the SM idle.)
    cudaFuncAttributes fa{};
    if ((e = cudaFuncGetAttributes(&fa, tmc::k_composite_tm<C, false, false>))) return e;
    int dev = 0, regs_sm = 0, smem_sm = 0, thr_sm = 0, blk_sm = 0, smem_rsv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    cudaDeviceGetAttribute(&blk_sm, cudaDevAttrMaxBlocksPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int regs_blk = ((fa.numRegs * 32 + 255) / 256 * 256) * (tmc::kThreads / 32);   // 256-register warp granules
    int per_sm = std::min(thr_sm / tmc::kThreads, blk_sm);
    per_sm = std::min(per_sm, regs_sm / std::max(1, regs_blk));
    per_sm = std::min(per_sm, smem_sm / (int)(smem + fa.sharedSizeBytes + smem_rsv));
    if (getenv("TA_DEBUG_PREP"))
        fprintf(stderr, "k_composite_tm<%d>: %d regs, smem %zu (+%d reserved), %d CTAs/SM before TMEM\n", C, fa.numRegs,
                smem, smem_rsv, per_sm);
    per_sm = std::min(per_sm, 512 / tmc::tmem_cols<C>());   // TMEM columns per SM
    if (cap > 0) per_sm = std::min(per_sm, cap);
    *resident = std::max(1, num_sms * std::max(1, per_sm));
    return cudaSuccess;
}

cudaError_t prepare_composite_tm(int num_sms, int ctas_per_sm_cap, int resident[4]) {
    cudaError_t e;
    resident[0] = 0;
    if ((e = prepare_tm_one<16>(num_sms, ctas_per_sm_cap, &resident[1])) ||
        (e = prepare_tm_one<32>(num_sms, ctas_per_sm_cap, &resident[2])) ||
        (e = prepare_tm_one<64>(num_sms, ctas_per_sm_cap, &resident[3])))
        return e;
    return cudaSuccess;
}

template <int C>
static cudaError_t launch_tm_c(int tiles, int resident, bool fast, const uint4* rec, const void* feat, const uint32_t* list,
                               const uint2* trng, const uint32_t* order, CompositeGeom cg, RasterConsts rc,
                               const CallState* cs, uint64_t list_cap, float* F, float* A, int32_t* ncontrib,
                               cudaStream_t st) {
    const size_t smem = sizeof(tmc::Smem<C>) + 1024;
    const int grid = std::min(tiles, resident);
    const __half* fh = static_cast<const __half*>(feat);
#define TA_TM(K, FA) tmc::k_composite_tm<C, K, FA><<<grid, tmc::kThreads, smem, st>>>(rec, fh, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib)
    if (ncontrib) {
        if (fast) TA_TM(true, true); else TA_TM(true, false);
    } else {
        if (fast) TA_TM(false, true); else TA_TM(false, false);
    }
#undef TA_TM
    return cudaGetLastError();
}

cudaError_t launch_composite_tm(int C, int tiles, const int* resident, bool fast, const uint4* rec, const void* feat,
                                const uint32_t* list, const uint2* trng, const uint32_t* order, CompositeGeom cg,
                                RasterConsts rc, const CallState* cs, uint64_t list_cap, float* F, float* A,
                                int32_t* ncontrib, cudaStream_t st) {
    switch (C) {
        case 16: return launch_tm_c<16>(tiles, resident[1], fast, rec, feat, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib, st);
        case 32: return launch_tm_c<32>(tiles, resident[2], fast, rec, feat, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib, st);
        case 64: return launch_tm_c<64>(tiles, resident[3], fast, rec, feat, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ta
