// composite_ws.cu -- warp-specialized compositor (sm_100a; fp16 features, C = 32, 16 x 16 tiles;
// opt-in TA_COMPOSITOR=3).
//
// The persistent compositor (composite.cu, k_composite_tc) alternates, in every warp, a fill phase
// (list read, splat-record gather, cull, staging) that waits on L2 latency with a compositing phase
// that is bound by the FP32 pipe.  Here each 8x8 block is served by a PAIR of warps: a producer warp
// runs the fill into one of two staging buffers while its consumer warp composites the other, so the
// gather latency overlaps the arithmetic of the same block instead of relying on other warps.  Per CTA:
// warps 0-3 produce, warps 4-7 consume (consumer 4+i owns TMEM lane quarter i for its 64 x 32
// accumulators, as in k_composite_tc's tensor-memory variant).  Buffers are handed over with one
// mbarrier per direction per buffer.  The consumer publishes the bounding box of its still-active
// pixels after each buffer; the producer culls against the latest one it sees for the block (it only
// shrinks, so a stale box is a conservative cull) and ends the block early once it is empty.  The
// recurrence, the decisions and the accumulation are those of k_composite_tc: the same bits of A and
// of the composited counts, F within fp32 summation grouping.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "internal.h"
#include "tc_dev.cuh"

namespace ta {
namespace wsc {

constexpr int C = 32;
constexpr int kProducers = 4;             // warpgroup 0
template <int kCPP>                       // consumers per producer: warpgroups 1 .. kCPP
constexpr int threads_for() { return 32 * kProducers * (1 + kCPP); }
#ifndef TA_WS_NB
#define TA_WS_NB 32
#endif
#ifndef TA_WS_BLOCKS
#define TA_WS_BLOCKS 3
#endif
// setmaxnreg rebalancing between the producer and consumer warpgroups (0: off)
#ifndef TA_WS_REGS_P
#define TA_WS_REGS_P 56
#endif
#ifndef TA_WS_REGS_C
#define TA_WS_REGS_C 104
#endif
// 1 producer : 2 consumers (TA_COMPOSITOR=4): 2 CTAs of 12 warps per SM, registers rebalanced
#ifndef TA_WS2_REGS_P
#define TA_WS2_REGS_P 48
#endif
#ifndef TA_WS2_REGS_C
#define TA_WS2_REGS_C 96
#endif
constexpr int NB = TA_WS_NB;              // entries per staging buffer
constexpr int PH = C + 8;                 // feature row pitch (halves): 5 x 16 B, an odd number of 16-B chunks
constexpr int WP = 36;                    // weight row pitch (words)
constexpr int NT = C / 8;
constexpr uint32_t kMtCols = C / 2;       // TMEM columns of one 16-pixel m-tile
constexpr int kFirst = 1, kLast = 2, kTerm = 4;

struct Stage {
    float4 p[NB / 2][4];                  // staged splat records, entry pairs interleaved (as k_composite_tc)
    __half f[NB][PH];                     // staged fp16 feature rows
    int cnt, flags, blk, pad;
};
struct Pair {
    Stage s[2];
    uint32_t w[2][16][WP];                // consumer: fp16 hi / lo weights of one 16-entry chunk
    int rblk, rect[4], pad[3];            // consumer -> producer: active-pixel box (x0, x1, y0, y1) of block rblk
    unsigned long long full[2], empty[2]; // mbarriers: buffer s filled / consumed
};
// A producer's walk through one consumer's current block (registers for 1 : 1, shared memory for 1 : 2)
struct FillState {
    uint32_t blk, pos, cend, pf_pos, pf0, pf1, fills0, fills1;
    int bx0, by0, ax0, ax1, ay0, ay1, first, active, term, s;
};

__device__ __forceinline__ bool mbar_test_parity(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n}\n" : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0u;
}

// One staging buffer of the producer's walk `fs` (the fill of k_composite_tc): list indices (one round
// ahead), splat records, cull against the consumer's latest active box, staging + feature rows by
// cp.async; then the header and the hand-over to the consumer.  Returns true after the block's last buffer.
template <bool kCounts>
__device__ __forceinline__ bool fill_one(FillState& fs, Pair& pr, const uint4* __restrict__ rec,
                                         const __half* __restrict__ feat, const uint32_t* __restrict__ clist, uint32_t n,
                                         float qlim, unsigned long long* wk) {
    const uint32_t lane = lane_id(), lt = lanemask_lt();
    const int s = fs.s;
    const uint32_t fills = s ? fs.fills1 : fs.fills0;
    if (fills) mbar_wait_parity_sleep(smem_u32(&pr.empty[s]), (fills - 1u) & 1u);
    if (!fs.first) {
        // lane 0 reads the consumer's latest box and the warp takes its copy (lanes reading separately
        // could see different publications, and the cull / fill below must be warp-uniform)
        int rb = 0, r0 = 0, r1 = 0, r2 = 0, r3 = 0;
        if (lane == 0) {
            rb = *(volatile int*)&pr.rblk;
            r0 = *(volatile int*)&pr.rect[0];
            r1 = *(volatile int*)&pr.rect[1];
            r2 = *(volatile int*)&pr.rect[2];
            r3 = *(volatile int*)&pr.rect[3];
        }
        rb = __shfl_sync(0xffffffffu, rb, 0);
        if (rb == (int)fs.blk) {
            fs.ax0 = __shfl_sync(0xffffffffu, r0, 0);
            fs.ax1 = __shfl_sync(0xffffffffu, r1, 0);
            fs.ay0 = __shfl_sync(0xffffffffu, r2, 0);
            fs.ay1 = __shfl_sync(0xffffffffu, r3, 0);
        }
    }
    Stage& st = pr.s[s];
    int cnt = 0;
    const int ax0 = fs.ax0, ax1 = fs.ax1, ay0 = fs.ay0, ay1 = fs.ay1, bx0 = fs.bx0, by0 = fs.by0;
    const uint32_t cend = fs.cend;
    uint32_t pos = fs.pos, pf_pos = fs.pf_pos, pf[2] = {fs.pf0, fs.pf1};
    const bool live = ax0 <= ax1 && ay0 <= ay1;
    if (live) {
        const float X0 = (float)ax0, X1 = (float)ax1, Y0 = (float)ay0, Y1 = (float)ay1;
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
                if (kp) {
                    const int d = cnt + (int)rank;
                    const int gx0 = (int)(r1[hh].z & 0xffff), gx1 = (int)(r1[hh].z >> 16);
                    const int gy0 = (int)(r1[hh].w & 0xffff), gy1 = (int)(r1[hh].w >> 16);
                    float* const pp = reinterpret_cast<float*>(&st.p[d >> 1][0]) + (d & 1);
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
                    const uint32_t dst = smem_u32(&st.f[d][0]);
#pragma unroll
                    for (int c = 0; c < C * 2; c += 16) cp_async16(dst + c, src + c);
                }
                cnt += __popc(bal);
                adv += step;
                if (step < 32u) break;
            }
            pos += adv;
            if (kCounts) { wk[0] += adv; wk[7] += 1; }
        }
    }
    cp_async_wait_all();
    const bool last = !live || pos >= cend;
    if (kCounts) wk[1] += cnt;
    if (lane == 0) { st.cnt = cnt; st.flags = (fs.first ? kFirst : 0) | (last ? kLast : 0); st.blk = (int)fs.blk; }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) mbar_arrive1(smem_u32(&pr.full[s]));
    if (s) fs.fills1++; else fs.fills0++;
    fs.s = s ^ 1;
    fs.first = 0;
    fs.pos = pos;
    fs.pf_pos = pf_pos;
    fs.pf0 = pf[0];
    fs.pf1 = pf[1];
    if (last) fs.active = 0;
    return last;
}

// Starts the producer's walk of the next block for a consumer (claims it); false when none is left.
__device__ __forceinline__ bool begin_block(FillState& fs, uint32_t* wq, uint32_t nblk, const uint32_t* __restrict__ order,
                                            const uint2* __restrict__ trng, const CompositeGeom& cg, uint64_t list_cap) {
    uint32_t blk = 0;
    if (lane_id() == 0) blk = atomicAdd(wq, 1u);
    blk = __shfl_sync(0xffffffffu, blk, 0);
    if (blk >= nblk) return false;
    const int tile = (int)order[blk >> 2];
    const uint32_t qd = blk & 3u;
    const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
    const uint2 tr = trng[tile];
    uint32_t cend = tr.x + tr.y;
    if (cend > list_cap) cend = (uint32_t)list_cap;
    fs.blk = blk;
    fs.pos = tr.x;
    fs.cend = cend;
    fs.pf_pos = 0xffffffffu;
    fs.bx0 = txi * kTile + 8 * (int)(qd & 1);
    fs.by0 = tyi * kTile + 8 * (int)(qd >> 1);
    // culling rectangle: the block's in-frame pixels until the consumer publishes its active box
    fs.ax0 = fs.bx0; fs.ax1 = min(fs.bx0 + 7, cg.W - 1);
    fs.ay0 = fs.by0; fs.ay1 = min(fs.by0 + 7, cg.H - 1);
    fs.first = 1;
    fs.active = 1;
    return true;
}

// Hands the terminate marker to a consumer through its next buffer.
__device__ __forceinline__ void send_term(FillState& fs, Pair& pr) {
    const int s = fs.s;
    const uint32_t fills = s ? fs.fills1 : fs.fills0;
    if (fills) mbar_wait_parity_sleep(smem_u32(&pr.empty[s]), (fills - 1u) & 1u);
    if (lane_id() == 0) { pr.s[s].cnt = 0; pr.s[s].flags = kTerm; pr.s[s].blk = -1; }
    __threadfence_block();
    __syncwarp();
    if (lane_id() == 0) mbar_arrive1(smem_u32(&pr.full[s]));
    fs.term = 1;
}

template <bool kCounts, bool kFast, int kCPP>
__global__ void __launch_bounds__(threads_for<kCPP>(), kCPP == 1 ? TA_WS_BLOCKS : 2)
k_composite_ws(const uint4* __restrict__ rec, const __half* __restrict__ feat, const uint32_t* __restrict__ clist,
               const uint2* __restrict__ trng, const uint32_t* __restrict__ order, CompositeGeom cg, RasterConsts rc,
               const CallState* __restrict__ cs, uint64_t list_cap, float* __restrict__ Fout, float* __restrict__ Aout,
               int32_t* __restrict__ ncontrib) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Pair* const pairs = reinterpret_cast<Pair*>(smem_raw);
    FillState* const pstate = reinterpret_cast<FillState*>(pairs + kProducers * kCPP);   // 1 : 2 walks
    __shared__ uint32_t s_tmem;
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const bool producer = warp < (uint32_t)kProducers;
    const int cidx = producer ? 0 : (int)warp - kProducers;        // consumer pair index
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "n"(64 * kCPP) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (producer && lane == 0) {
        for (int c = 0; c < kCPP; c++) {
            Pair& q = pairs[(int)warp + kProducers * c];
            for (int k = 0; k < 2; k++) { mbar_init1(smem_u32(&q.full[k])); mbar_init1(smem_u32(&q.empty[k])); }
            q.rblk = -1;
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int W = cg.W, H = cg.H;
    const uint32_t nblk = 4u * (uint32_t)(cg.TX * cg.TY);
    unsigned long long wk[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    if (producer) {
        // ================================================================ producer: fill
        if (kCPP == 1) { if (TA_WS_REGS_P) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TA_WS_REGS_P)); }
        else { if (TA_WS2_REGS_P) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TA_WS2_REGS_P)); }
        uint32_t* const wq = &const_cast<CallState*>(cs)->scan_counter[6];
        const uint32_t n = cs->n;
        const float qlim = rc.q_max * 1.015625f + 0.01f;
        if (kCPP == 1) {
            Pair& pr = pairs[warp];
            FillState fs;
            fs.fills0 = fs.fills1 = 0u;
            fs.s = 0;
            fs.term = 0;
            for (;;) {
                if (!begin_block(fs, wq, nblk, order, trng, cg, list_cap)) { send_term(fs, pr); break; }
                if (kCounts) wk[6] += 1;
                while (!fill_one<kCounts>(fs, pr, rec, feat, clist, n, qlim, wk)) {}
            }
        } else {
            // one producer, kCPP consumers: serve whichever consumer has a free buffer; walks in shared memory
            FillState* const my = pstate + (int)warp * kCPP;
            if (lane == 0)
                for (int c = 0; c < kCPP; c++) {
                    my[c].fills0 = my[c].fills1 = 0u;
                    my[c].s = 0;
                    my[c].term = 0;
                    my[c].active = 0;
                }
            __syncwarp();
            for (;;) {
                bool all_done = true, progressed = false;
                for (int c = 0; c < kCPP; c++) {
                    FillState fs = my[c];
                    if (fs.term) continue;
                    all_done = false;
                    Pair& pr = pairs[(int)warp + kProducers * c];
                    const uint32_t fills = fs.s ? fs.fills1 : fs.fills0;
                    // (one lane's view of the barrier for the whole warp: lanes polling separately could
                    //  disagree while the phase completes, and the fill below is warp-synchronous)
                    const bool free_buf = !fills || __shfl_sync(0xffffffffu, (uint32_t)mbar_test_parity(
                                                       smem_u32(&pr.empty[fs.s]), (fills - 1u) & 1u), 0) != 0u;
                    if (!free_buf) continue;
                    progressed = true;
                    if (!fs.active) {
                        if (!begin_block(fs, wq, nblk, order, trng, cg, list_cap)) {
                            send_term(fs, pr);
                            __syncwarp();
                            if (lane == 0) my[c] = fs;
                            __syncwarp();
                            continue;
                        }
                        if (kCounts) wk[6] += 1;
                    }
                    fill_one<kCounts>(fs, pr, rec, feat, clist, n, qlim, wk);
                    fs.pf_pos = 0xffffffffu;        // the prefetched indices are per lane: not kept in the shared walk
                    __syncwarp();
                    if (lane == 0) my[c] = fs;
                    __syncwarp();
                }
                if (all_done) break;
                if (!progressed) __nanosleep(256);
            }
        }
    } else {
        Pair& pr = pairs[cidx];
        // ================================================================ consumer: composite
        if (kCPP == 1) { if (TA_WS_REGS_C) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TA_WS_REGS_C)); }
        else { if (TA_WS2_REGS_C) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TA_WS2_REGS_C)); }
        const uint32_t tacc = s_tmem + ((32u * (warp & 3u)) << 16) + 64u * (uint32_t)(cidx / kProducers);
        const float teps = rc.t_eps, qlo = rc.q_lo_half, amx = rc.a_max_2k, alo = rc.a_min_2k;
        const int li = (int)lane;
        const uint32_t a_base = smem_u32(&pr.w[0][(li & 7) + 8 * (li >> 4)][0]) + (uint32_t)(((li >> 3) & 1) * 16);
        constexpr uint32_t kLoOff = 16 * WP * 4;
        const int bk = (li & 7) + 8 * ((li >> 3) & 1);
        uint32_t* const wst = &pr.w[0][0][li];
        uint32_t uses[2] = {0u, 0u};
        int s = 0;
        // per-block state (set when a block's first buffer arrives)
        int bx0 = 0, by0 = 0, px = 0, pyA = 0, pyB = 0;
        float pxf = 0.0f;
        float2 py2 = make_float2(0.0f, 0.0f);
        float2 T = make_float2(1.0f, 1.0f);
        int ncA = 0, ncB = 0;
        uint32_t actA = 0u, actB = 0u;
        bool modeB = false, movedA = false, movedB = false, chas = false;
        int ol = 0, hs = 0, cpx = 0, cpy = 0, nc1 = 0;
        float T1 = 1.0f;
        uint32_t act1 = 0u;
        for (;;) {
            mbar_wait_parity_sleep(smem_u32(&pr.full[s]), uses[s] & 1u);
            Stage& st = pr.s[s];
            const int cnt = st.cnt, flags = st.flags, blk = st.blk;
            if (flags & kTerm) break;
            if (flags & kFirst) {
                const int tile = (int)order[(uint32_t)blk >> 2];
                const uint32_t qd = (uint32_t)blk & 3u;
                const int tyi = tile / cg.TX, txi = tile - tyi * cg.TX;
                bx0 = txi * kTile + 8 * (int)(qd & 1);
                by0 = tyi * kTile + 8 * (int)(qd >> 1);
                px = bx0 + (int)(lane & 7);
                pyA = by0 + (int)(lane >> 3);
                pyB = pyA + 4;
                pxf = (float)px;
                py2 = make_float2((float)pyA, (float)pyB);
                T = make_float2(1.0f, 1.0f);
                ncA = ncB = 0;
                actA = (px < W && pyA < H) ? (1u << lane) : 0u;
                actB = (px < W && pyB < H) ? (1u << lane) : 0u;
                modeB = movedA = movedB = chas = false;
                ol = hs = cpx = cpy = nc1 = 0;
                T1 = 1.0f;
                act1 = 0u;
                float z[16];
#pragma unroll
                for (int i = 0; i < 16; i++) z[i] = 0.0f;
#pragma unroll
                for (int mt = 0; mt < 4; mt++) tm_st16(tacc + kMtCols * mt, z);
            }
            const uint32_t b_base = smem_u32(&st.f[0][0]) + (uint32_t)((li >> 4) * 16);
            if (__any_sync(0xffffffffu, (actA | actB | act1) != 0u)) {
                for (int j0 = 0; j0 < cnt; j0 += 16) {
                    const int nk = min(16, cnt - j0);
                    if (!modeB) {
                        const uint32_t mA = __ballot_sync(0xffffffffu, actA != 0u), mB = __ballot_sync(0xffffffffu, actB != 0u);
                        const int nA = __popc(mA), na = nA + __popc(mB);
                        if (na <= 32) {                           // the compacted mode of k_composite_tc
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
                            uint4* wz = reinterpret_cast<uint4*>(&pr.w[0][0][0]);
                            for (int k = li; k < 2 * 16 * WP / 4; k += 32) wz[k] = make_uint4(0u, 0u, 0u, 0u);
                            __syncwarp();
                        }
                    }
                    if (modeB) {
                        const float cpxf = (float)cpx, cpyf = (float)cpy;
                        __half* const wh = reinterpret_cast<__half*>(&pr.w[0][0][0]) + 2 * ol + hs;
#pragma unroll 2
                        for (int jj = 0; jj < 16; jj += 2) {
                            float w0 = 0.0f, w1 = 0.0f;
                            if (jj < nk) {
                                const bool has1 = jj + 1 < nk;
                                const float4* const pq = st.p[(j0 + jj) >> 1];
                                const float4 P0 = pq[0], P1 = pq[1], P2 = pq[2], P3 = pq[3];
                                const float2 dx = sub2(bc2(cpxf), make_float2(P0.x, P0.y));
                                const float2 dy = sub2(bc2(cpyf), make_float2(P0.z, P0.w));
                                const float2 t1 = mul2(make_float2(P1.z, P1.w), dy);
                                const float2 t2 = fma2(make_float2(P1.x, P1.y), dx, t1);
                                const float2 t4 = mul2(mul2(make_float2(P2.x, P2.y), dy), dy);
                                const float2 q = fma2(t2, dx, t4);
                                const uint32_t b0 = __float_as_uint(hs ? P3.z : P3.x), b1 = __float_as_uint(hs ? P3.w : P3.y);
                                const float qm0 = (act1 && ((b0 >> ol) & 1u)) ? q.x : -kInf;
                                const float qm1 = (act1 && has1 && ((b1 >> ol) & 1u)) ? q.y : -kInf;
                                if (kCounts) wk[2] += has1 ? 2 : 1;
                                const float2 e = exp2v<kFast>(q);
                                const float2 ae = mul2(make_float2(P2.z, P2.w), e);
                                const float2 a = make_float2(fminf(amx, ae.x), fminf(amx, ae.y));
                                const float2 om = fma2(a, bc2(-1.0f / 2048.0f), bc2(1.0f));
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
                        auto pairs_loop = [&](auto full) {
                            constexpr bool kFull = decltype(full)::value;
#pragma unroll
                            for (int jj = 0; jj < 16; jj += 2) {
                                float2 w0 = make_float2(0.0f, 0.0f), w1 = make_float2(0.0f, 0.0f);
                                if (kFull || jj < nk) {
                                    const float4* const pq = st.p[(j0 + jj) >> 1];
                                    const float4 P0 = pq[0], P1 = pq[1], P2 = pq[2], P3 = pq[3];
                                    const float4 G0 = make_float4(P0.x, P0.z, P1.x, P1.z), G1 = make_float4(P0.y, P0.w, P1.y, P1.w);
                                    const float4 H0 = make_float4(P2.x, P2.z, P3.x, P3.z), H1 = make_float4(P2.y, P2.w, P3.y, P3.w);
                                    const float2 q0 = quad_q(G0, H0.x, pxf, py2), q1 = quad_q(G1, H1.x, pxf, py2);
                                    const uint32_t mA0 = __float_as_uint(H0.z), mB0 = __float_as_uint(H0.w);
                                    const bool has1 = kFull || jj + 1 < nk;
                                    const uint32_t mA1 = has1 ? __float_as_uint(H1.z) : 0u, mB1 = has1 ? __float_as_uint(H1.w) : 0u;
                                    if (kCounts) wk[2] += has1 ? 2 : 1;
                                    const float2 x0 = exp2v<kFast>(q0);
                                    const float2 x1 = exp2v<kFast>(q1);
                                    const float2 ae0 = mul2(bc2(H0.y), x0), ae1 = mul2(bc2(H1.y), x1);
                                    const float2 a0 = make_float2(fminf(amx, ae0.x), fminf(amx, ae0.y));
                                    const float2 a1 = make_float2(fminf(amx, ae1.x), fminf(amx, ae1.y));
                                    if (kCounts) {
                                        wk[3] += __any_sync(0xffffffffu, ((mA0 & actA) && q0.x >= qlo) || ((mB0 & actB) && q0.y >= qlo)) ? 1 : 0;
                                        wk[3] += __any_sync(0xffffffffu, ((mA1 & actA) && q1.x >= qlo) || ((mB1 & actB) && q1.y >= qlo)) ? 1 : 0;
                                    }
                                    w0 = tstep<kCounts>(q0, a0, mA0, mB0, qlo, alo, teps, T, actA, actB, ncA, ncB, wk);
                                    w1 = tstep<kCounts>(q1, a1, mA1, mB1, qlo, alo, teps, T, actA, actB, ncA, ncB, wk);
                                }
                                const __half2 h0 = __floats2half2_rn(w0.x, w0.y), h1 = __floats2half2_rn(w1.x, w1.y);
                                const float2 r0 = sub2(w0, __half22float2(h0)), r1 = sub2(w1, __half22float2(h1));
                                const __half2 l0 = __floats2half2_rn(r0.x, r0.y), l1 = __floats2half2_rn(r1.x, r1.y);
                                wst[jj * WP] = *reinterpret_cast<const uint32_t*>(&h0);
                                wst[(jj + 1) * WP] = *reinterpret_cast<const uint32_t*>(&h1);
                                wst[16 * WP + jj * WP] = *reinterpret_cast<const uint32_t*>(&l0);
                                wst[16 * WP + (jj + 1) * WP] = *reinterpret_cast<const uint32_t*>(&l1);
                            }
                        };
                        if (nk == 16) pairs_loop(std::integral_constant<bool, true>());
                        else pairs_loop(std::integral_constant<bool, false>());
                    }
                    __syncwarp();
                    uint32_t bfr[NT][2];
                    {
                        const int row = min(j0 + bk, cnt - 1);
                        const uint32_t rb = b_base + (uint32_t)(row * PH * 2);
#pragma unroll
                        for (int np = 0; np < NT / 2; np++)
                            ldsm_x4_t(rb + np * 32, bfr[2 * np][0], bfr[2 * np][1], bfr[2 * np + 1][0], bfr[2 * np + 1][1]);
                    }
                    tm_wait_st();
#pragma unroll
                    for (int mt = 0; mt < 4; mt++) {
                        uint32_t ah[4], al[4];
                        ldsm_x4_t(a_base + mt * 32, ah[0], ah[1], ah[2], ah[3]);
                        ldsm_x4_t(a_base + mt * 32 + kLoOff, al[0], al[1], al[2], al[3]);
                        float v[16];
                        tm_ld16(tacc + kMtCols * mt, v);
                        float (&am)[NT][4] = *reinterpret_cast<float (*)[NT][4]>(v);
#pragma unroll
                        for (int nt = 0; nt < NT; nt++) {
                            hmma16816(am[nt], ah, bfr[nt][0], bfr[nt][1]);
                            hmma16816(am[nt], al, bfr[nt][0], bfr[nt][1]);
                        }
                        tm_st16(tacc + kMtCols * mt, v);
                    }
                    __syncwarp();
                    if (!__any_sync(0xffffffffu, (actA | actB | act1) != 0u)) break;
                }
            }
            // publish the bounding box of the pixels still compositing (empty once all stopped)
            {
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
                const int ax0 = __reduce_min_sync(0xffffffffu, lx0), ax1 = __reduce_max_sync(0xffffffffu, lx1);
                const int ay0 = __reduce_min_sync(0xffffffffu, ly0), ay1 = __reduce_max_sync(0xffffffffu, ly1);
                if (lane == 0) {
                    *(volatile int*)&pr.rect[0] = ax0;
                    *(volatile int*)&pr.rect[1] = ax1;
                    *(volatile int*)&pr.rect[2] = ay0;
                    *(volatile int*)&pr.rect[3] = ay1;
                    __threadfence_block();
                    *(volatile int*)&pr.rblk = blk;
                }
            }
            if (flags & kLast) {
                // write the block: F from tensor memory (fragment layout of k_composite_tc), A, counts
                const int g = li >> 2, t = li & 3;
                tm_wait_st();
#pragma unroll
                for (int mt = 0; mt < 4; mt++) {
                    float tv[16];
                    tm_ld16(tacc + kMtCols * mt, tv);
                    float (&acm)[NT][4] = *reinterpret_cast<float (*)[NT][4]>(tv);
#pragma unroll
                    for (int half = 0; half < 2; half++) {
                        const int r = g + 8 * half;
                        const int l2 = 8 * mt + (r >> 1);
                        const int ox = bx0 + (l2 & 7), oy = by0 + (l2 >> 3) + 4 * (r & 1);
                        if (ox < W && oy < H) {
                            float* out = Fout + ((size_t)oy * W + ox) * C + 2 * t;
#pragma unroll
                            for (int nt = 0; nt < NT; nt++)
                                *reinterpret_cast<float2*>(out + 8 * nt) =
                                    make_float2(acm[nt][2 * half] * (1.0f / 2048.0f), acm[nt][2 * half + 1] * (1.0f / 2048.0f));
                        }
                    }
                }
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const int py = hh ? pyB : pyA;
                    if (px < W && py < H && !(hh ? movedB : movedA)) {
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
            __syncwarp();
            if (lane == 0) mbar_arrive1(smem_u32(&pr.empty[s]));
            uses[s]++;
            s ^= 1;
        }
    }
    if (kCounts && lane == 0) {
        unsigned long long* work = const_cast<CallState*>(cs)->work;
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (wk[k]) atomicAdd(&work[k], wk[k]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(64 * kCPP) : "memory");
}

}  // namespace wsc

// Per-device preparation: shared-memory opt-in and co-resident CTAs (registers, shared memory, TMEM).
template <int kCPP>
static size_t ws_smem() { return sizeof(wsc::Pair) * wsc::kProducers * kCPP + (kCPP > 1 ? sizeof(wsc::FillState) * wsc::kProducers * kCPP : 0); }

template <int kCPP>
static cudaError_t prepare_ws(int num_sms, int cap, int* resident) {
    const int smem = (int)ws_smem<kCPP>();
    const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(wsc::k_composite_ws<false, false, kCPP>, A, smem)) ||
        (e = cudaFuncSetAttribute(wsc::k_composite_ws<true, false, kCPP>, A, smem)) ||
        (e = cudaFuncSetAttribute(wsc::k_composite_ws<false, true, kCPP>, A, smem)) ||
        (e = cudaFuncSetAttribute(wsc::k_composite_ws<true, true, kCPP>, A, smem)))
        return e;
    cudaFuncAttributes fa{};
    if ((e = cudaFuncGetAttributes(&fa, wsc::k_composite_ws<false, false, kCPP>))) return e;
    int dev = 0, regs_sm = 0, smem_sm = 0, thr_sm = 0, blk_sm = 0, smem_rsv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    cudaDeviceGetAttribute(&blk_sm, cudaDevAttrMaxBlocksPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    constexpr int kThr = wsc::threads_for<kCPP>();
    const int regs_blk = ((fa.numRegs * 32 + 255) / 256 * 256) * (kThr / 32);
    int per_sm = std::min(thr_sm / kThr, blk_sm);
    per_sm = std::min(per_sm, regs_sm / std::max(1, regs_blk));
    per_sm = std::min(per_sm, smem_sm / (smem + (int)fa.sharedSizeBytes + smem_rsv));
    per_sm = std::min(per_sm, 512 / (64 * kCPP));
    if (getenv("TA_DEBUG_PREP"))
        fprintf(stderr, "k_composite_ws<1:%d>: %d regs, %d B local, smem %d, %d CTAs/SM\n", kCPP, fa.numRegs,
                (int)fa.localSizeBytes, smem, per_sm);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    *resident = std::max(1, num_sms * std::max(1, per_sm));
    return cudaSuccess;
}

cudaError_t prepare_composite_ws(int num_sms, int cap, int* resident) {
    cudaError_t e;
    if ((e = prepare_ws<1>(num_sms, cap, &resident[0])) || (e = prepare_ws<2>(num_sms, cap, &resident[1]))) return e;
    return cudaSuccess;
}

template <int kCPP>
static cudaError_t launch_ws(int tiles, int resident, bool fast, const uint4* rec, const void* feat, const uint32_t* list,
                             const uint2* trng, uint32_t* order, CompositeGeom cg, RasterConsts rc, const CallState* cs,
                             uint64_t list_cap, float* F, float* A, int32_t* ncontrib, cudaStream_t st) {
    const size_t smem = ws_smem<kCPP>();
    const int grid = std::min(tiles, resident);
    constexpr int kThr = wsc::threads_for<kCPP>();
    const __half* fh = static_cast<const __half*>(feat);
#define TA_WS(K, FA) wsc::k_composite_ws<K, FA, kCPP><<<grid, kThr, smem, st>>>(rec, fh, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib)
    if (ncontrib) {
        if (fast) TA_WS(true, true); else TA_WS(true, false);
    } else {
        if (fast) TA_WS(false, true); else TA_WS(false, false);
    }
#undef TA_WS
    return cudaGetLastError();
}

cudaError_t launch_composite_ws(int cpp, int tiles, const int* resident, bool fast, const uint4* rec, const void* feat,
                                const uint32_t* list, const uint2* trng, uint32_t* order, CompositeGeom cg, RasterConsts rc,
                                const CallState* cs, uint64_t list_cap, float* F, float* A, int32_t* ncontrib,
                                cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    launch_tile_order(trng, cg, order, st);
    return cpp == 2 ? launch_ws<2>(tiles, resident[1], fast, rec, feat, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib, st)
                    : launch_ws<1>(tiles, resident[0], fast, rec, feat, list, trng, order, cg, rc, cs, list_cap, F, A, ncontrib, st);
}

}  // namespace ta
