// api.cu -- the C ABI of include/ta.h: validation, scratch management, kernel orchestration.
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include "../../include/ta.h"
#include "common.cuh"
#include "internal.h"

using namespace ta;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// Scans per rasterize call: depth-sort passes 0..3 use status regions / counters 0..3, the
// tile-offset scan uses 4.
constexpr int kScanSlots = 6;   // + slot 5: debug tile-list scan

}  // namespace

struct ta_context {
    int device = 0;
    int num_sms = 148;
    size_t smem_optin = 0;
    // per-context launch configuration (ta_context_create, on this context's device): persistent grid
    // sizes of the compositor / backward per C slot, and the tuning knobs read once from the environment
    int resident_ws[2] = {1, 1};  // warp-specialized compositor (TA_COMPOSITOR=3: 1 producer : 1 consumer, 4: 1 : 2)
    int resident_tc[6] = {1, 1, 1, 1, 1, 1}, resident_bwd[4] = {1, 1, 1, 1}, resident_tm[4] = {0, 1, 1, 1};
    int compositor = 0;           // TA_COMPOSITOR: 0 = mma.sync persistent-warp kernel (default; for fp16 C = 32 / 64 with
                                  // its accumulators in tensor memory), 1 = register (+ shared) accumulators for every C,
                                  // 2 = tensor-memory MMA kernel (tcgen05.mma, fp16 C >= 16; measured slower),
                                  // 3 / 4 = warp-specialized producer : consumer = 1 : 1 / 1 : 2 (fp16 C = 32;
                                  // measured slower)
    int coarse64_above = 1024;    // TA_COARSE64_ABOVE: 64-px coarse bins for targets wider / taller than this
    int tile_px = 16;             // TA_TILE_PX=8: 8 x 8 compositing tiles under 32-px coarse bins (opt-in, measured
                                  // slower: DESIGN.md section 6); 64-px bins and the TMEM compositor always use 16
    bool bwd_simt = false;        // TA_BWD_SIMT: force the plain backward kernel
    std::string err;
    uint64_t launches = 0;
    DevBuf cs, status, rec, boxes, tile_order, keys0, keys1, vals0, vals1, sort_hist, bin_offs, list, ncontrib, ucounts, ustatus;
    DevBuf tlist, trng;           // per-tile lists (tiles-per-bin x the coarse-list capacity) and their (start, count)
    DevBuf zkey;                  // ta_zbuffer: 64-bit z-buffer words
    DevBuf ffeat, frec, fkey, fval, fstats, fn;   // fused front end: compact features, per-target records / keys
    // fused front end, targets 1..T-1: child contexts (own scratch) + streams, so the targets' sort / bin /
    // composite chains run concurrently after the shared front end
    ta_context* aux[kMaxFrontTargets - 1] = {nullptr, nullptr, nullptr};
    cudaStream_t aux_stream[kMaxFrontTargets - 1] = {nullptr, nullptr, nullptr};
    cudaEvent_t aux_ev[kMaxFrontTargets] = {nullptr, nullptr, nullptr, nullptr};
    int64_t rsv_g = -1, rsv_e = 0;  // the last ta_reserve (applied to child contexts created later)
    int32_t rsv_H = 0, rsv_W = 0;
    uint64_t* pinned = nullptr;
    uint32_t status_region = 0;   // words per scan slot
    // last rasterize call
    bool have_last = false;
    int last_TX = 0, last_TY = 0, last_H = 0, last_W = 0;
    uint32_t last_P = 0;
    bool last_counts = false;
    CompositeGeom last_cg{};
    int last_C = 0, last_fbytes = 0;  // the forward call the backward pass must match
    int64_t last_n = 0;
    const void* last_feat = nullptr;
    RasterConsts last_rc{};
    const void* last_rec = nullptr;           // the arrays the last call's debug view reads
    const void* last_k[2] = {nullptr, nullptr};
    const void* last_v[2] = {nullptr, nullptr};
    DevBuf dbg_offs, dbg_list;
    // stage profiling
    bool profiling = false;
    struct EvPair { cudaEvent_t a, b; int stage; };
    std::vector<EvPair> pending, pool;
    double prof_ms[TA_STAGE_COUNT] = {0};
    uint64_t prof_calls[TA_STAGE_COUNT] = {0};
};

namespace {

ta_status fail(ta_context* c, ta_status s, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return s;
}

ta_status cuda_fail(ta_context* c, cudaError_t e, const char* where) {
    return fail(c, TA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define TA_CUDA(ctx, expr)                                          \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return cuda_fail((ctx), _e, #expr); \
    } while (0)

#define TA_LAUNCHED(ctx)                                                    \
    do {                                                                    \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess) return cuda_fail((ctx), _e, "kernel launch"); \
        (ctx)->launches++;                                                  \
    } while (0)

ta_status grow(ta_context* c, DevBuf& b, size_t bytes) {
    if (bytes <= b.bytes) return TA_OK;
    if (b.p) {
        cudaError_t e = cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaFree");
    }
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        return fail(c, TA_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
    }
    b.bytes = want;
    return TA_OK;
}

bool finite_cam(const ta_intrinsics& K, const ta_extrinsics& RT, ta_context* c, ta_status* st) {
    const float* v = &K.fx;
    for (int i = 0; i < 4; i++)
        if (!std::isfinite(v[i])) { *st = fail(c, TA_ERR_INVALID_ARG, "non-finite intrinsics"); return false; }
    if (!(K.fx > 0.0f) || !(K.fy > 0.0f)) { *st = fail(c, TA_ERR_INVALID_ARG, "fx, fy must be > 0"); return false; }
    for (int i = 0; i < 9; i++)
        if (!std::isfinite(RT.R[i])) { *st = fail(c, TA_ERR_INVALID_ARG, "non-finite rotation"); return false; }
    for (int i = 0; i < 3; i++)
        if (!std::isfinite(RT.t[i])) { *st = fail(c, TA_ERR_INVALID_ARG, "non-finite translation"); return false; }
    double worst = 0.0;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double d = 0.0;
            for (int k = 0; k < 3; k++) d += (double)RT.R[i * 3 + k] * (double)RT.R[j * 3 + k];
            worst = std::max(worst, std::fabs(d - (i == j ? 1.0 : 0.0)));
        }
    const float* R = RT.R;
    const double det = (double)R[0] * ((double)R[4] * R[8] - (double)R[5] * R[7]) -
                       (double)R[1] * ((double)R[3] * R[8] - (double)R[5] * R[6]) +
                       (double)R[2] * ((double)R[3] * R[7] - (double)R[4] * R[6]);
    if (worst > 1e-4 || det <= 0.0) {
        *st = fail(c, TA_ERR_INVALID_ARG, "rotation not orthonormal (|R R^T - I| = %g, det %g)", worst, det);
        return false;
    }
    return true;
}

bool supported_C(int C) { return C == 8 || C == 16 || C == 32 || C == 64; }

// Stage timer: records an event pair around a stage when profiling is enabled.
struct StageTimer {
    ta_context* c;
    cudaStream_t s;
    ta_context::EvPair cur{};
    bool on = false;
    StageTimer(ta_context* c_, cudaStream_t s_) : c(c_), s(s_) {}
    void begin(int stage) {
        if (!c->profiling) return;
        if (c->pool.empty()) {
            ta_context::EvPair p{};
            cudaEventCreate(&p.a);
            cudaEventCreate(&p.b);
            c->pool.push_back(p);
        }
        cur = c->pool.back();
        c->pool.pop_back();
        cur.stage = stage;
        cudaEventRecord(cur.a, s);
        on = true;
    }
    void end() {
        if (!on) return;
        cudaEventRecord(cur.b, s);
        c->pending.push_back(cur);
        on = false;
    }
};

}  // namespace

extern "C" {

void ta_default_params(ta_raster_params* p) {
    if (!p) return;
    p->dilation = 0.3f;
    p->alpha_max = 0.99f;
    p->alpha_min = 1.0f / 255.0f;
    p->t_eps = 1e-4f;
    p->cull_sigma = 3.0f;
    p->z_near = 0.01f;
    p->d_min = 0.0f;
    p->default_scale = 0.0f;
    p->default_opacity = 1.0f;
    p->flags = 0u;
    p->exact_exp = 1;
}

const char* ta_status_string(ta_status s) {
    switch (s) {
        case TA_OK: return "TA_OK";
        case TA_ERR_INVALID_ARG: return "TA_ERR_INVALID_ARG";
        case TA_ERR_UNSUPPORTED: return "TA_ERR_UNSUPPORTED";
        case TA_ERR_CUDA: return "TA_ERR_CUDA";
        case TA_ERR_OUT_OF_MEMORY: return "TA_ERR_OUT_OF_MEMORY";
        case TA_ERR_CAPACITY: return "TA_ERR_CAPACITY";
    }
    return "TA_ERR_UNKNOWN";
}

const char* ta_last_error(const ta_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

const char* ta_build_info(void) {
    return "taloha sm_100a (persistent-warp compositor: packed-fp32 recurrence + mma.sync f16 feature accumulation into tensor-memory accumulators; one-sweep depth sort; look-back scans; coarse binning + tile split; tensor-core backward)";
}

uint64_t ta_launch_count(const ta_context* ctx) {
    if (!ctx) return 0;
    uint64_t n = ctx->launches;
    for (int k = 0; k < kMaxFrontTargets - 1; k++)
        if (ctx->aux[k]) n += ctx->aux[k]->launches;
    return n;
}

ta_status ta_context_create(int32_t device, ta_context** out) {
    if (!out) return TA_ERR_INVALID_ARG;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) { cudaGetLastError(); return TA_ERR_CUDA; }
    if (device < 0 || device >= ndev) return TA_ERR_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return TA_ERR_CUDA;
    ta_context* c = new ta_context();
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c->smem_optin = (size_t)optin;
    ta_status st = grow(c, c->cs, sizeof(CallState));
    if (st != TA_OK) { delete c; return st; }
    if (cudaMemset(c->cs.p, 0, sizeof(CallState)) != cudaSuccess ||
        cudaMallocHost(&c->pinned, 64) != cudaSuccess ||
        cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) != cudaSuccess ||
        cudaFuncSetAttribute(k_bin_place, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) != cudaSuccess) {
        cudaGetLastError();
        if (c->pinned) cudaFreeHost(c->pinned);
        cudaFree(c->cs.p);
        delete c;
        return TA_ERR_CUDA;
    }
    if (const char* e = getenv("TA_COARSE64_ABOVE")) c->coarse64_above = atoi(e);   // tuning knobs
    if (const char* e = getenv("TA_TILE_PX")) c->tile_px = atoi(e) == 8 ? 8 : 16;
    c->bwd_simt = getenv("TA_BWD_SIMT") != nullptr;
    const int cap = getenv("TA_TC_CTAS_PER_SM") ? atoi(getenv("TA_TC_CTAS_PER_SM")) : 0;
    if (const char* e = getenv("TA_COMPOSITOR")) c->compositor = atoi(e);
    const int cap_tm = getenv("TA_TM_CTAS_PER_SM") ? atoi(getenv("TA_TM_CTAS_PER_SM")) : 0;
    if (prepare_composite(c->num_sms, cap, c->resident_tc) != cudaSuccess ||
        prepare_composite_tm(c->num_sms, cap_tm, c->resident_tm) != cudaSuccess ||
        prepare_composite_ws(c->num_sms, cap, c->resident_ws) != cudaSuccess ||
        prepare_composite_bwd(c->num_sms, c->resident_bwd) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeHost(c->pinned);
        cudaFree(c->cs.p);
        delete c;
        return TA_ERR_CUDA;
    }
    *out = c;
    return TA_OK;
}

ta_status ta_context_destroy(ta_context* c) {
    if (!c) return TA_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    DevBuf* bufs[] = {&c->cs, &c->status, &c->rec, &c->boxes, &c->tile_order, &c->keys0, &c->keys1, &c->vals0, &c->vals1, &c->sort_hist,
                      &c->bin_offs, &c->list, &c->ncontrib, &c->ucounts, &c->ustatus, &c->dbg_offs, &c->dbg_list,
                      &c->tlist, &c->trng, &c->zkey, &c->ffeat, &c->frec, &c->fkey, &c->fval, &c->fstats, &c->fn};
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    if (c->pinned) cudaFreeHost(c->pinned);
    for (int k = 0; k < kMaxFrontTargets - 1; k++) {
        if (c->aux[k]) ta_context_destroy(c->aux[k]);
        if (c->aux_stream[k]) cudaStreamDestroy(c->aux_stream[k]);
    }
    for (int k = 0; k < kMaxFrontTargets; k++)
        if (c->aux_ev[k]) cudaEventDestroy(c->aux_ev[k]);
    for (auto& p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto& p : c->pool) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    delete c;
    return TA_OK;
}

}  // extern "C"

namespace {

// Coarse-binning geometry for an H x W target and up to cap Gaussians: 32 x 32-pixel bins up to 1024
// pixels on a side, 64 x 64 beyond when the Gaussian indices fit the 24 index bits of such bins' list
// entries (keeps the bin count, and with it the per-warp shared-memory cursors of k_bin_place, at
// ~1024 for 2048^2), warps per binning block (per-warp [NB] cursors + lane masks must fit in shared
// memory), P = rank tiles of nw * 256 ranks.  Compositing tiles: 16 x 16 pixels; opt-in (TA_TILE_PX=8)
// 8 x 8 under 32-pixel bins (4 x 4 tiles per bin, 24 index bits), where each compositor warp walks a
// list holding only the Gaussians whose box reaches its own 8 x 8 block (c3: 38 % fewer list entries
// read, compositor -6.5 %, but 2.9x the tile entries and +0.15 ms of tile split: slower per view).
ta_status bin_geometry(ta_context* c, int H, int W, int64_t cap, BinGeom* bg) {
    const int min_side6 = c->coarse64_above;
    bg->shift = (std::max(H, W) > min_side6 && cap <= ((int64_t)1 << entry_idx_bits(kMaxCoarseShift - 4))) ? kMaxCoarseShift : 5;
    if (cap > ((int64_t)1 << entry_idx_bits(1)))
        return fail(c, TA_ERR_CAPACITY, "more than 2^%d Gaussians", entry_idx_bits(1));
    bg->ts = (bg->shift == 5 && c->tile_px == 8 && c->compositor != 2 && cap <= ((int64_t)1 << entry_idx_bits(2))) ? 3 : 4;
    const int bs = 1 << bg->shift;
    bg->TX = (W + bs - 1) / bs;
    bg->TY = (H + bs - 1) / bs;
    const int NB = bg->TX * bg->TY;
    const size_t per_warp = (size_t)NB * 8;      // write cursors + lane masks
    const size_t budget = c->smem_optin > 4096 ? c->smem_optin - 1024 : 0;
    int w = (int)std::min<size_t>(8, budget / per_warp);
    if (w < 1) return fail(c, TA_ERR_UNSUPPORTED, "target of %d x %d coarse bins exceeds the binning shared-memory budget",
                           bg->TX, bg->TY);
    bg->nw = w;
    const uint64_t R = kBinTileRanks(w);
    bg->P = (uint32_t)(((uint64_t)std::max<int64_t>(cap, 1) + R - 1) / R);
    return TA_OK;
}

// tiles per coarse bin
inline uint64_t tiles_per_bin(const BinGeom& bg) { return 1ull << (2 * (bg.shift - bg.ts)); }

CompositeGeom composite_geometry(const BinGeom& bg, int H, int W) {
    CompositeGeom cg;
    const int tp = 1 << bg.ts;
    cg.TX = (W + tp - 1) / tp;
    cg.TY = (H + tp - 1) / tp;
    cg.ts = bg.ts;
    cg.W = W;
    cg.H = H;
    cg.shift = bg.shift;
    cg.BX = bg.TX;
    cg.P = bg.P;
    return cg;
}

// Coarse list (entries x 4 B) and the per-tile lists (tiles per bin x 4 B).  Per-tile list positions
// are 32-bit (trng, the compositors' cursors), so the tile-list space nq x entries must stay below 2^32.
ta_status reserve_lists(ta_context* c, size_t entries, const BinGeom& bg) {
    ta_status st;
    const size_t nq = (size_t)tiles_per_bin(bg);
    entries = std::max<size_t>(entries, 1);
    if ((uint64_t)entries * nq > 0xffffffffull)
        return fail(c, TA_ERR_CAPACITY, "%zu coarse entries x %zu tiles per bin exceed the 2^32-1 tile-list positions",
                    entries, nq);
    if ((st = grow(c, c->list, entries * 4)) != TA_OK) return st;
    return grow(c, c->tlist, entries * 4 * nq);
}

bool lists_reserved(const ta_context* c, size_t entries, const BinGeom& bg) {
    const size_t nq = (size_t)tiles_per_bin(bg);
    return c->list.bytes >= entries * 4 && c->tlist.bytes >= entries * 4 * nq;
}

ta_status reserve_gaussians(ta_context* c, int64_t cap) {
    ta_status st;
    const size_t n = (size_t)std::max<int64_t>(cap, 1);
    if ((st = grow(c, c->rec, n * 32)) != TA_OK) return st;
    if ((st = grow(c, c->boxes, n * 8)) != TA_OK) return st;
    if ((st = grow(c, c->keys0, n * 4)) != TA_OK) return st;
    if ((st = grow(c, c->keys1, n * 4)) != TA_OK) return st;
    if ((st = grow(c, c->vals0, n * 4)) != TA_OK) return st;
    if ((st = grow(c, c->vals1, n * 4)) != TA_OK) return st;
    const size_t parts = (n + kSortKeysPerBlock - 1) / kSortKeysPerBlock;
    const size_t lb_bytes = 4 * 256 * parts * 8;       // depth-sort look-back words, 4 passes
    if (c->sort_hist.bytes < lb_bytes) {
        if ((st = grow(c, c->sort_hist, lb_bytes)) != TA_OK) return st;
        if (cudaMemset(c->sort_hist.p, 0, c->sort_hist.bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
            return fail(c, TA_ERR_CUDA, "cudaMemset");
    }
    return TA_OK;
}

ta_status reserve_target(ta_context* c, const BinGeom& bg, int64_t cap, int H, int W) {
    ta_status st;
    const size_t T = (size_t)bg.TX * bg.TY;
    const size_t bin_len = T * bg.P + 1;
    if ((st = grow(c, c->bin_offs, bin_len * 4 + 64)) != TA_OK) return st;
    {
        const CompositeGeom cg0 = composite_geometry(bg, H, W);
        if ((st = grow(c, c->tile_order, (size_t)cg0.TX * cg0.TY * 4 + 64)) != TA_OK) return st;
        if ((st = grow(c, c->trng, (size_t)cg0.TX * cg0.TY * 8 + 64)) != TA_OK) return st;
    }
    const size_t parts = ((size_t)std::max<int64_t>(cap, 1) + kSortKeysPerBlock - 1) / kSortKeysPerBlock;
    const CompositeGeom cg = composite_geometry(bg, H, W);
    const uint32_t region = std::max(std::max(scan_tiles((uint32_t)(256 * parts)), scan_tiles((uint32_t)bin_len)),
                                     scan_tiles((uint32_t)(cg.TX * cg.TY) + 1));
    if (region > c->status_region || !c->status.p) {
        if ((st = grow(c, c->status, (size_t)region * kScanSlots * 8)) != TA_OK) return st;
        c->status_region = region;
    }
    return TA_OK;
}

// Validates V source views and fills the kernels' view table (unprojection-block ranges, running
// pixel offsets, 128-bit-load eligibility).  need_feat: the views must carry 16-byte aligned features.
ta_status build_view_table(ta_context* c, const ta_source_view* views, int32_t V, const ta_raster_params* p,
                           bool need_feat, int C, int fbytes, ViewTable* vtp, int64_t* pixels_out, uint32_t* blocks_out) {
    ViewTable& vt = *vtp;
    memset(&vt, 0, sizeof(vt));
    vt.V = V;
    vt.C = C;
    vt.fbytes = fbytes;
    vt.d_min = p->d_min;
    vt.default_scale = p->default_scale;
    vt.default_opacity = p->default_opacity;
    int64_t pixels = 0;
    uint32_t blocks = 0;
    for (int v = 0; v < V; v++) {
        const ta_source_view& s = views[v];
        if (s.H < 1 || s.W < 1 || s.H > 32767 || s.W > 32767)
            return fail(c, TA_ERR_INVALID_ARG, "view %d: bad size %d x %d", v, s.H, s.W);
        if (!s.disparity || (need_feat && !s.feat)) return fail(c, TA_ERR_INVALID_ARG, "view %d: NULL disparity/feat", v);
        if (!(s.baseline > 0.0f) || !std::isfinite(s.baseline))
            return fail(c, TA_ERR_INVALID_ARG, "view %d: baseline must be > 0", v);
        ta_status cst;
        if (!finite_cam(s.K, s.RT, c, &cst)) return cst;
        if (need_feat && (((uintptr_t)s.feat) & 15)) return fail(c, TA_ERR_INVALID_ARG, "view %d: feat not 16-byte aligned", v);
        ViewDesc& d = vt.v[v];
        d.disp = s.disparity; d.mask = s.mask; d.scale = s.scale; d.quat = s.quat; d.opacity = s.opacity; d.feat = s.feat;
        d.fx = s.K.fx; d.fy = s.K.fy; d.cx = s.K.cx; d.cy = s.K.cy;
        memcpy(d.R, s.RT.R, sizeof(d.R));
        memcpy(d.t, s.RT.t, sizeof(d.t));
        d.baseline = s.baseline;
        d.H = s.H; d.W = s.W;
        d.blk_begin = blocks;
        d.idx0 = (uint32_t)pixels;
        const int64_t HW = (int64_t)s.H * s.W;
        const bool al = ((((uintptr_t)s.disparity) | ((uintptr_t)s.opacity) | ((uintptr_t)s.quat)) & 15) == 0 &&
                        (((uintptr_t)s.mask) & 3) == 0;
        d.vec4 = (HW % 4 == 0 && al) ? 1 : 0;
        blocks += (uint32_t)((HW + kUnprojPix - 1) / kUnprojPix);
        pixels += HW;
    }
    *pixels_out = pixels;
    *blocks_out = blocks;
    return TA_OK;
}

void fill_cam(const ta_intrinsics& K, const ta_extrinsics& RT, int H, int W, TargetCam* cam) {
    cam->fx = K.fx; cam->fy = K.fy; cam->cx = K.cx; cam->cy = K.cy;
    memcpy(cam->R, RT.R, sizeof(cam->R));
    memcpy(cam->t, RT.t, sizeof(cam->t));
    cam->W = W; cam->H = H;
    cam->Wm1f = (float)(W - 1);
    cam->Hm1f = (float)(H - 1);
}

void fill_consts(const ta_raster_params& p, RasterConsts* rc) {
    rc->dilation = p.dilation; rc->alpha_max = p.alpha_max; rc->alpha_min = p.alpha_min; rc->t_eps = p.t_eps;
    rc->cull_sigma = p.cull_sigma; rc->z_near = p.z_near;
    rc->q_max = p.cull_sigma * p.cull_sigma;
    rc->q_lo_half = -0.5f * rc->q_max;
    rc->a_max_2k = 2048.0f * p.alpha_max;
    rc->a_min_2k = 2048.0f * p.alpha_min;
}

// One rasterization (a2 -- a6) of a Gaussian set into one target.  Gaussian-set mode (pos_alpha / cov
// given): k_project writes the splat records into context scratch.  Pre-projected mode (rec / k0 / v0 /
// stats given, from the fused front end): the records, depth keys and visibility statistics exist
// already and the pipeline starts at the depth sort.
struct RasterJob {
    const float4* pos_alpha = nullptr;
    const float4* cov = nullptr;
    uint4* rec = nullptr;
    uint32_t* k0 = nullptr;
    uint32_t* v0 = nullptr;
    const uint32_t* stats = nullptr;
    const void* feat = nullptr;
    int C = 0, fbytes = 2;
    int64_t n = -1;                    // host count or -1 (read n_dev on the device)
    const int64_t* n_dev = nullptr;
    int64_t cap = 0;                   // upper bound on n (scratch sizing)
    TargetCam cam{};
    RasterConsts rc{};
    int H = 0, W = 0;
    bool async = false, counts = false, fast_exp = false;
    float* F = nullptr;
    float* A = nullptr;
    cudaStream_t s = nullptr;
};

ta_status raster_pipeline(ta_context* c, const RasterJob& job);

// Child contexts (own scratch) + non-blocking streams for lanes 1..L-1 of the multi-target calls, and
// the events that fork from / join into the caller's stream.  A reservation made on the parent is
// applied to children created later.
ta_status ensure_lanes(ta_context* c, int L) {
    for (int k = 1; k < L; k++) {
        if (!c->aux[k - 1]) {
            ta_status cst = ta_context_create(c->device, &c->aux[k - 1]);
            if (cst != TA_OK) return fail(c, cst, "child context %d", k);
            c->aux[k - 1]->compositor = c->compositor;
            if (cudaStreamCreateWithFlags(&c->aux_stream[k - 1], cudaStreamNonBlocking) != cudaSuccess)
                return fail(c, TA_ERR_CUDA, "child stream %d", k);
            if (c->rsv_g >= 0 && (cst = ta_reserve(c->aux[k - 1], c->rsv_g, c->rsv_e, c->rsv_H, c->rsv_W)) != TA_OK)
                return fail(c, cst, "child reserve: %s", c->aux[k - 1]->err.c_str());
        }
    }
    for (int k = 0; k < L; k++)
        if (!c->aux_ev[k] && cudaEventCreateWithFlags(&c->aux_ev[k], cudaEventDisableTiming) != cudaSuccess)
            return fail(c, TA_ERR_CUDA, "lane event");
    return TA_OK;
}

bool params_ok(const ta_raster_params& p) {
    return (p.cull_sigma > 0.0f && p.cull_sigma <= 12.0f) && (p.alpha_max > 0.0f && p.alpha_max < 1.0f) &&
           (p.t_eps > 0.0f && p.t_eps < 1.0f) && (p.alpha_min >= 0.0f) && (p.dilation >= 0.0f) && std::isfinite(p.z_near);
}

}  // namespace

extern "C" {

ta_status ta_reserve(ta_context* c, int64_t max_gaussians, int64_t max_entries, int32_t H, int32_t W) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (max_gaussians < 0 || max_entries < 0 || H <= 0 || W <= 0 || H > 32767 || W > 32767)
        return fail(c, TA_ERR_INVALID_ARG, "ta_reserve: bad sizes");
    if (max_entries > 0xffffffffll) return fail(c, TA_ERR_CAPACITY, "more than 2^32-1 tile entries");   // (and reserve_lists:
                                                                                                        //  x tiles per bin)
    cudaSetDevice(c->device);
    ta_status st;
    if ((st = reserve_gaussians(c, max_gaussians)) != TA_OK) return st;
    BinGeom bg;
    if ((st = bin_geometry(c, H, W, max_gaussians, &bg)) != TA_OK) return st;
    if ((st = reserve_target(c, bg, max_gaussians, H, W)) != TA_OK) return st;
    if ((st = reserve_lists(c, (size_t)std::max<int64_t>(max_entries, 1), bg)) != TA_OK) return st;
    c->rsv_g = max_gaussians; c->rsv_e = max_entries; c->rsv_H = H; c->rsv_W = W;
    for (int k = 0; k < kMaxFrontTargets - 1; k++)
        if (c->aux[k] && (st = ta_reserve(c->aux[k], max_gaussians, max_entries, H, W)) != TA_OK)
            return fail(c, st, "child context: %s", c->aux[k]->err.c_str());
    return TA_OK;
}

ta_status ta_unproject(ta_context* c, const ta_source_view* views, int32_t V, const ta_raster_params* p,
                       ta_gaussians* out, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!views || !p || !out) return fail(c, TA_ERR_INVALID_ARG, "ta_unproject: NULL argument");
    if (V < 1 || V > TA_MAX_VIEWS) return fail(c, TA_ERR_UNSUPPORTED, "ta_unproject: V = %d not in [1, %d]", V, TA_MAX_VIEWS);
    if (!supported_C(out->C)) return fail(c, TA_ERR_UNSUPPORTED, "C = %d not in {8,16,32,64}", out->C);
    if (out->feat_dtype != TA_F32 && out->feat_dtype != TA_F16) return fail(c, TA_ERR_UNSUPPORTED, "unknown dtype");
    if (!out->pos_alpha || !out->cov || !out->feat || !out->n_dev)
        return fail(c, TA_ERR_INVALID_ARG, "ta_unproject: NULL output array");
    if ((((uintptr_t)out->pos_alpha) | ((uintptr_t)out->cov) | ((uintptr_t)out->feat)) & 15)
        return fail(c, TA_ERR_INVALID_ARG, "Gaussian arrays must be 16-byte aligned");
    cudaSetDevice(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    ViewTable vt;
    int64_t pixels = 0;
    uint32_t blocks = 0;
    ta_status vst = build_view_table(c, views, V, p, true, out->C, out->feat_dtype == TA_F16 ? 2 : 4, &vt, &pixels, &blocks);
    if (vst != TA_OK) return vst;
    if (pixels > out->capacity)
        return fail(c, TA_ERR_CAPACITY, "capacity %lld < %lld source pixels", (long long)out->capacity, (long long)pixels);
    if (pixels >= (1ll << 31)) return fail(c, TA_ERR_CAPACITY, "more than 2^31 source pixels");
    ta_status s2;
    if ((s2 = grow(c, c->ucounts, ((size_t)blocks + 16) * 4)) != TA_OK) return s2;
    const uint32_t tiles = scan_tiles(blocks);
    if ((s2 = grow(c, c->ustatus, ((size_t)tiles + 8) * 8)) != TA_OK) return s2;
    StageTimer tm(c, st);
    tm.begin(TA_STAGE_UNPROJECT);
    TA_CUDA(c, cudaMemsetAsync(c->ustatus.p, 0, ((size_t)tiles + 8) * 8, st));
    k_unproject_count<<<blocks, kUnprojThreads, 0, st>>>(vt, (uint32_t*)c->ucounts.p);
    TA_LAUNCHED(c);
    unsigned long long* status = (unsigned long long*)c->ustatus.p;
    launch_scan((uint32_t*)c->ucounts.p, nullptr, blocks, status, (uint32_t*)(status + tiles + 4),
                (unsigned long long*)out->n_dev, st);
    TA_LAUNCHED(c);
    k_unproject_write<<<blocks, kUnprojThreads, 0, st>>>(vt, (const uint32_t*)c->ucounts.p, (float4*)out->pos_alpha,
                                                         (float4*)out->cov, out->feat);
    TA_LAUNCHED(c);
    tm.end();
    return TA_OK;
}

ta_status ta_rasterize(ta_context* c, const ta_gaussians* g, int64_t n, const ta_intrinsics* K,
                       const ta_extrinsics* RT, int32_t H, int32_t W, const ta_raster_params* p, float* feat_out,
                       float* alpha_out, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!g || !K || !RT || !p || !feat_out || !alpha_out) return fail(c, TA_ERR_INVALID_ARG, "ta_rasterize: NULL argument");
    if (H < 1 || W < 1 || H > 32767 || W > 32767) return fail(c, TA_ERR_INVALID_ARG, "bad target size %d x %d", H, W);
    if (!supported_C(g->C)) return fail(c, TA_ERR_UNSUPPORTED, "C = %d not in {8,16,32,64}", g->C);
    if (g->feat_dtype != TA_F32 && g->feat_dtype != TA_F16) return fail(c, TA_ERR_UNSUPPORTED, "unknown dtype");
    if (n < -1 || (n == -1 && !g->n_dev)) return fail(c, TA_ERR_INVALID_ARG, "n = -1 needs g->n_dev");
    if (n > g->capacity) return fail(c, TA_ERR_INVALID_ARG, "n > capacity");
    if ((n != 0) && (!g->pos_alpha || !g->cov || !g->feat)) return fail(c, TA_ERR_INVALID_ARG, "NULL Gaussian array");
    if ((((uintptr_t)g->pos_alpha) | ((uintptr_t)g->cov) | ((uintptr_t)g->feat) | ((uintptr_t)feat_out)) & 15)
        return fail(c, TA_ERR_INVALID_ARG, "Gaussian arrays / feat_out must be 16-byte aligned");
    if (!(p->cull_sigma > 0.0f && p->cull_sigma <= 12.0f) || !(p->alpha_max > 0.0f && p->alpha_max < 1.0f) ||
        !(p->t_eps > 0.0f && p->t_eps < 1.0f) || !(p->alpha_min >= 0.0f) || !(p->dilation >= 0.0f) ||
        !std::isfinite(p->z_near))
        return fail(c, TA_ERR_INVALID_ARG, "raster params out of range (0 < cull_sigma <= 12, 0 < alpha_max < 1, "
                                           "0 < t_eps < 1, alpha_min >= 0, dilation >= 0)");
    ta_status st;
    if (!finite_cam(*K, *RT, c, &st)) return st;
    cudaSetDevice(c->device);
    RasterJob job;
    job.pos_alpha = (const float4*)g->pos_alpha;
    job.cov = (const float4*)g->cov;
    job.feat = g->feat;
    job.C = g->C;
    job.fbytes = g->feat_dtype == TA_F16 ? 2 : 4;
    job.n = n;
    job.n_dev = g->n_dev;
    job.cap = n >= 0 ? n : g->capacity;
    job.H = H; job.W = W;
    fill_cam(*K, *RT, H, W, &job.cam);
    fill_consts(*p, &job.rc);
    if (p->exact_exp != 0 && p->exact_exp != 1) return fail(c, TA_ERR_INVALID_ARG, "exact_exp must be 0 or 1");
    job.fast_exp = p->exact_exp == 0;
    job.async = (p->flags & TA_FLAG_ASYNC) != 0;
    job.counts = (p->flags & TA_FLAG_DEBUG_COUNTS) != 0;
    job.F = feat_out; job.A = alpha_out;
    job.s = (cudaStream_t)stream;
    return raster_pipeline(c, job);
}

}  // extern "C"

namespace {

ta_status raster_pipeline(ta_context* c, const RasterJob& job) {
    ta_status st;
    const int64_t cap = job.cap, n = job.n;
    const int H = job.H, W = job.W;
    const bool async = job.async, counts = job.counts, fast_exp = job.fast_exp;
    const TargetCam& cam = job.cam;
    const RasterConsts& rc = job.rc;
    cudaStream_t s = job.s;
    float* feat_out = job.F;
    float* alpha_out = job.A;
    BinGeom bg;
    if ((st = bin_geometry(c, H, W, cap, &bg)) != TA_OK) return st;
    const int NB = bg.TX * bg.TY;                      // coarse bins
    const uint32_t bin_len = (uint32_t)NB * bg.P + 1;
    const CompositeGeom cg = composite_geometry(bg, H, W);
    const int T = cg.TX * cg.TY;                       // compositing tiles
    if (async) {
        if (c->rec.bytes < (size_t)cap * 32 || c->bin_offs.bytes < (size_t)bin_len * 4 || !c->list.p ||
            !lists_reserved(c, c->list.bytes / 4, bg))
            return fail(c, TA_ERR_CAPACITY, "TA_FLAG_ASYNC needs ta_reserve() for this size first");
    }
    if ((st = reserve_gaussians(c, cap)) != TA_OK) return st;
    if ((st = reserve_target(c, bg, cap, H, W)) != TA_OK) return st;
    if (counts && (st = grow(c, c->ncontrib, (size_t)H * W * 4)) != TA_OK) return st;
    {
        const uint64_t nq = tiles_per_bin(bg);
        const uint64_t first = std::min<uint64_t>((uint64_t)std::max<int64_t>(cap, 1) * 4, 0xffffffffull / nq);
        if ((st = reserve_lists(c, c->list.p ? std::min<uint64_t>(c->list.bytes / 4, 0xffffffffull / nq) : first,
                                bg)) != TA_OK)
            return st;
    }


    CallState* cs = (CallState*)c->cs.p;
    unsigned long long* status = (unsigned long long*)c->status.p;
    const uint32_t region = c->status_region;
    const int n_status = (int)(region * kScanSlots);
    const bool pre = job.rec != nullptr;
    uint32_t* k0 = pre ? job.k0 : (uint32_t*)c->keys0.p; uint32_t* k1 = (uint32_t*)c->keys1.p;
    uint32_t* v0 = pre ? job.v0 : (uint32_t*)c->vals0.p; uint32_t* v1 = (uint32_t*)c->vals1.p;
    unsigned long long* sort_lb = (unsigned long long*)c->sort_hist.p;
    uint32_t* offs = (uint32_t*)c->bin_offs.p;
    uint4* rec = pre ? job.rec : (uint4*)c->rec.p;

    StageTimer tm(c, s);
    tm.begin(TA_STAGE_PROJECT);
    k_init<<<std::min(1024, (n_status + 255) / 256 + 1), 256, 0, s>>>(cs, status, n_status, n, job.n_dev,
                                                                       kBinTileRanks(bg.nw), (uint32_t)NB, job.stats);
    TA_LAUNCHED(c);
    const int64_t cap_blocks = (cap + 255) / 256;
    if (cap_blocks > 0 && !pre) {
        k_project<<<(unsigned)((cap + 511) / 512), 256, 0, s>>>(job.pos_alpha, job.cov, cam, rc, cs, rec, k0, v0);
        TA_LAUNCHED(c);
    }
    tm.end();
    tm.begin(TA_STAGE_SORT);
    const uint32_t parts_max = (uint32_t)((cap + kSortKeysPerBlock - 1) / kSortKeysPerBlock);
    const uint32_t sort_blocks = parts_max;
    if (sort_blocks > 0) {
        k_sort_digits<<<(unsigned)std::min<int64_t>((cap + 2047) / 2048, 2 * c->num_sms), 256, 0, s>>>(k0, cs);
        TA_LAUNCHED(c);
        for (int pass = 0; pass < 4; pass++) {
            k_sort_pass<<<sort_blocks, kSortWarps * 32, 0, s>>>(k0, k1, v0, v1, pass, cs,
                                                                sort_lb + (size_t)pass * 256 * parts_max, rec,
                                                                (uint2*)c->boxes.p);
            TA_LAUNCHED(c);
        }
    }
    tm.end();
    const size_t smem_count = (size_t)NB * 4;
    const size_t smem_place = (size_t)bg.nw * NB * 8;
    tm.begin(TA_STAGE_BIN_COUNT);
    if (cap_blocks > 0) {
        k_gather_boxes<<<(unsigned)std::min<int64_t>(cap_blocks, 2 * c->num_sms), 256, 0, s>>>(rec, v0, v1, cs,
                                                                                            (uint2*)c->boxes.p);
        TA_LAUNCHED(c);
    }
    k_bin_count<<<bg.P, bg.nw * 32, smem_count, s>>>((const uint2*)c->boxes.p, cs, bg, offs);
    TA_LAUNCHED(c);
    tm.end();
    tm.begin(TA_STAGE_BIN_SCAN);
    launch_scan(offs, &cs->bin_len, bin_len, status + (size_t)4 * region, &cs->scan_counter[4], &cs->K, s);
    TA_LAUNCHED(c);
    if (!async) {
        TA_CUDA(c, cudaMemcpyAsync(c->pinned, &cs->K, 8, cudaMemcpyDeviceToHost, s));
        TA_CUDA(c, cudaStreamSynchronize(s));
        const uint64_t Kh = c->pinned[0];
        const uint64_t nq = tiles_per_bin(bg);
        if (Kh * nq > 0xffffffffull)
            return fail(c, TA_ERR_CAPACITY, "%llu coarse entries x %llu tiles per bin exceed 2^32-1 tile-list positions",
                        (unsigned long long)Kh, (unsigned long long)nq);
        if (!lists_reserved(c, (size_t)Kh, bg)) {
            // grow by 1/8 headroom, but never past the 32-bit tile-list position space
            const uint64_t want = std::min<uint64_t>(std::max<uint64_t>(c->list.bytes / 4, Kh + Kh / 8 + 1024),
                                                     0xffffffffull / nq);
            if ((st = reserve_lists(c, (size_t)want, bg)) != TA_OK) return st;
        }
    }
    tm.end();
    tm.begin(TA_STAGE_BIN_PLACE);
    k_bin_place<<<bg.P, bg.nw * 32, smem_place, s>>>((const uint2*)c->boxes.p, v0, v1, cs, bg, offs, (uint32_t*)c->list.p,
                                                     (uint64_t)(c->list.bytes / 4));
    TA_LAUNCHED(c);
    launch_tile_split((const uint32_t*)c->list.p, offs, cg, cs, (uint64_t)(c->list.bytes / 4), (uint32_t*)c->tlist.p,
                      (uint64_t)(c->tlist.bytes / 4), (uint2*)c->trng.p, s);
    TA_LAUNCHED(c);
    tm.end();
    tm.begin(TA_STAGE_COMPOSITE);
    cudaError_t e;
    if (job.fbytes == 2 && job.C >= 16 && c->compositor == 2) {
        // tensor-memory compositor (tcgen05.mma, accumulators in TMEM); exact_exp = 0 selects its SFU exp
        if (T > 0) launch_tile_order((const uint2*)c->trng.p, cg, (uint32_t*)c->tile_order.p, s);
        e = T > 0 ? launch_composite_tm(job.C, T, c->resident_tm, fast_exp, rec, job.feat, (const uint32_t*)c->tlist.p,
                                        (const uint2*)c->trng.p, (const uint32_t*)c->tile_order.p, cg, rc, cs,
                                        (uint64_t)(c->tlist.bytes / 4), feat_out, alpha_out,
                                        counts ? (int32_t*)c->ncontrib.p : nullptr, s)
                  : cudaSuccess;
    } else if (job.fbytes == 2 && job.C == 32 && (c->compositor == 3 || c->compositor == 4) && cg.ts == 4) {
        // warp-specialized compositor: producer (fill) / consumer (composite) warps, 1 : 1 or 1 : 2
        e = launch_composite_ws(c->compositor == 4 ? 2 : 1, T, c->resident_ws, fast_exp, rec, job.feat, (const uint32_t*)c->tlist.p,
                                (const uint2*)c->trng.p, (uint32_t*)c->tile_order.p, cg, rc, cs,
                                (uint64_t)(c->tlist.bytes / 4), feat_out, alpha_out,
                                counts ? (int32_t*)c->ncontrib.p : nullptr, s);
    } else {
        // persistent-warp compositors: mma.sync (fp16 features) / SIMT (fp32 features)
        e = launch_composite(job.C, job.fbytes, T, c->resident_tc, fast_exp, rec, job.feat,
                             (const uint32_t*)c->tlist.p, (const uint2*)c->trng.p, (uint32_t*)c->tile_order.p, cg, rc, cs,
                             (uint64_t)(c->tlist.bytes / 4), feat_out, alpha_out,
                             counts ? (int32_t*)c->ncontrib.p : nullptr, s, c->compositor == 0);
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "composite launch");
    c->launches += 2;   // k_tile_order + k_composite
    tm.end();
    c->have_last = true;
    c->last_TX = cg.TX; c->last_TY = cg.TY; c->last_P = bg.P; c->last_H = H; c->last_W = W;
    c->last_cg = cg;
    c->last_counts = counts;
    c->last_C = job.C;
    c->last_fbytes = job.fbytes;
    c->last_n = n;
    c->last_feat = job.feat;
    c->last_rc = rc;
    c->last_rec = rec;
    c->last_k[0] = k0; c->last_k[1] = k1;
    c->last_v[0] = v0; c->last_v[1] = v1;
    return TA_OK;
}

}  // namespace

extern "C" {


ta_status ta_rasterize_views(ta_context* c, const ta_gaussians* g, int64_t n, int32_t T, const ta_intrinsics* K_tgt,
                            const ta_extrinsics* RT_tgt, int32_t H, int32_t W, const ta_raster_params* p,
                            float* const* feat_out, float* const* alpha_out, int32_t lanes, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!g || !K_tgt || !RT_tgt || !p || !feat_out || !alpha_out)
        return fail(c, TA_ERR_INVALID_ARG, "ta_rasterize_views: NULL argument");
    if (T < 1) return fail(c, TA_ERR_INVALID_ARG, "T = %d < 1", T);
    if (lanes < 1 || lanes > kMaxFrontTargets) return fail(c, TA_ERR_INVALID_ARG, "lanes = %d not in [1, %d]", lanes, kMaxFrontTargets);
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int L = std::min<int>(lanes, T);
    ta_status st;
    if ((st = ensure_lanes(c, L)) != TA_OK) return st;
    if (L > 1) {
        TA_CUDA(c, cudaEventRecord(c->aux_ev[0], s));
        for (int k = 1; k < L; k++) TA_CUDA(c, cudaStreamWaitEvent(c->aux_stream[k - 1], c->aux_ev[0], 0));
    }
    for (int t = 0; t < T; t++) {                  // targets round-robin over the lanes, in order per lane
        const int k = t % L;
        ta_context* ct = k == 0 ? c : c->aux[k - 1];
        st = ta_rasterize(ct, g, n, &K_tgt[t], &RT_tgt[t], H, W, p, feat_out[t], alpha_out[t],
                          k == 0 ? stream : (void*)c->aux_stream[k - 1]);
        if (st != TA_OK) return ct == c ? st : fail(c, st, "target %d: %s", t, ct->err.c_str());
    }
    for (int k = 1; k < L; k++) {                  // the call completes on `stream`
        TA_CUDA(c, cudaEventRecord(c->aux_ev[k], c->aux_stream[k - 1]));
        TA_CUDA(c, cudaStreamWaitEvent(s, c->aux_ev[k], 0));
    }
    return TA_OK;
}

ta_status ta_render_sources(ta_context* c, const ta_source_view* views, int32_t V, int32_t C, ta_dtype feat_dtype,
                            const ta_raster_params* p, int32_t T, const ta_intrinsics* K_tgt, const ta_extrinsics* RT_tgt,
                            int32_t H, int32_t W, float* const* feat_out, float* const* alpha_out, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!views || !p || !K_tgt || !RT_tgt || !feat_out || !alpha_out)
        return fail(c, TA_ERR_INVALID_ARG, "ta_render_sources: NULL argument");
    if (V < 1 || V > TA_MAX_VIEWS) return fail(c, TA_ERR_UNSUPPORTED, "ta_render_sources: V = %d not in [1, %d]", V, TA_MAX_VIEWS);
    if (T < 1 || T > kMaxFrontTargets) return fail(c, TA_ERR_INVALID_ARG, "T = %d not in [1, %d]", T, kMaxFrontTargets);
    if (!supported_C(C)) return fail(c, TA_ERR_UNSUPPORTED, "C = %d not in {8,16,32,64}", C);
    if (feat_dtype != TA_F32 && feat_dtype != TA_F16) return fail(c, TA_ERR_UNSUPPORTED, "unknown dtype");
    if (H < 1 || W < 1 || H > 32767 || W > 32767) return fail(c, TA_ERR_INVALID_ARG, "bad target size %d x %d", H, W);
    if (!params_ok(*p))
        return fail(c, TA_ERR_INVALID_ARG, "raster params out of range (0 < cull_sigma <= 12, 0 < alpha_max < 1, "
                                           "0 < t_eps < 1, alpha_min >= 0, dilation >= 0)");
    if (p->exact_exp != 0 && p->exact_exp != 1) return fail(c, TA_ERR_INVALID_ARG, "exact_exp must be 0 or 1");
    ta_status st;
    for (int t = 0; t < T; t++) {
        if (!feat_out[t] || !alpha_out[t]) return fail(c, TA_ERR_INVALID_ARG, "target %d: NULL output", t);
        if (((uintptr_t)feat_out[t]) & 15) return fail(c, TA_ERR_INVALID_ARG, "target %d: feat_out not 16-byte aligned", t);
        if (!finite_cam(K_tgt[t], RT_tgt[t], c, &st)) return st;
    }
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int fbytes = feat_dtype == TA_F16 ? 2 : 4;
    ViewTable vt;
    int64_t pixels = 0;
    uint32_t blocks = 0;
    if ((st = build_view_table(c, views, V, p, true, C, fbytes, &vt, &pixels, &blocks)) != TA_OK) return st;
    if (pixels >= (1ll << 31)) return fail(c, TA_ERR_CAPACITY, "more than 2^31 source pixels");
    const size_t cap = (size_t)std::max<int64_t>(pixels, 1);
    if ((st = grow(c, c->ucounts, ((size_t)blocks + 16) * 4)) != TA_OK) return st;
    const uint32_t tiles = scan_tiles(blocks);
    if ((st = grow(c, c->ustatus, ((size_t)tiles + 8) * 8)) != TA_OK) return st;
    if ((st = grow(c, c->ffeat, cap * (size_t)C * fbytes)) != TA_OK ||
        (st = grow(c, c->frec, cap * 32 * (size_t)T)) != TA_OK || (st = grow(c, c->fkey, cap * 4 * (size_t)T)) != TA_OK ||
        (st = grow(c, c->fval, cap * 4 * (size_t)T)) != TA_OK || (st = grow(c, c->fstats, 16 * 4 * kMaxFrontTargets)) != TA_OK ||
        (st = grow(c, c->fn, 64)) != TA_OK)
        return st;
    RasterConsts rc;
    fill_consts(*p, &rc);
    FrontTargets ft;
    memset(&ft, 0, sizeof(ft));
    ft.T = T;
    for (int t = 0; t < T; t++) {
        fill_cam(K_tgt[t], RT_tgt[t], H, W, &ft.cam[t]);
        ft.rec[t] = (uint4*)c->frec.p + 2 * cap * t;
        ft.key[t] = (uint32_t*)c->fkey.p + cap * t;
        ft.val[t] = (uint32_t*)c->fval.p + cap * t;
    }
    uint32_t* stats = (uint32_t*)c->fstats.p;
    int64_t* n_dev = (int64_t*)c->fn.p;
    StageTimer tm(c, s);
    tm.begin(TA_STAGE_PROJECT);
    TA_CUDA(c, cudaMemsetAsync(c->ustatus.p, 0, ((size_t)tiles + 8) * 8, s));
    k_front_stats_init<<<1, 32, 0, s>>>(stats, T);
    TA_LAUNCHED(c);
    k_unproject_count<<<blocks, kUnprojThreads, 0, s>>>(vt, (uint32_t*)c->ucounts.p);
    TA_LAUNCHED(c);
    unsigned long long* ust = (unsigned long long*)c->ustatus.p;
    launch_scan((uint32_t*)c->ucounts.p, nullptr, blocks, ust, (uint32_t*)(ust + tiles + 4), (unsigned long long*)n_dev, s);
    TA_LAUNCHED(c);
    k_front_fused<<<blocks, kUnprojThreads, 0, s>>>(vt, (const uint32_t*)c->ucounts.p, ft, rc, c->ffeat.p, stats);
    TA_LAUNCHED(c);
    tm.end();
    // targets 1..T-1 run on child contexts / streams concurrently with target 0 (after the front end)
    if ((st = ensure_lanes(c, T)) != TA_OK) return st;
    if (T > 1) {
        TA_CUDA(c, cudaEventRecord(c->aux_ev[0], s));
        for (int t = 1; t < T; t++) TA_CUDA(c, cudaStreamWaitEvent(c->aux_stream[t - 1], c->aux_ev[0], 0));
    }
    for (int t = 0; t < T; t++) {
        ta_context* ct = t == 0 ? c : c->aux[t - 1];
        ct->profiling = c->profiling && t == 0;
        RasterJob job;
        job.rec = ft.rec[t];
        job.k0 = ft.key[t];
        job.v0 = ft.val[t];
        job.stats = stats + 3 * t;
        job.feat = c->ffeat.p;
        job.C = C;
        job.fbytes = fbytes;
        job.n = -1;
        job.n_dev = n_dev;
        job.cap = (int64_t)cap;
        job.cam = ft.cam[t];
        job.rc = rc;
        job.H = H; job.W = W;
        job.fast_exp = p->exact_exp == 0;
        job.async = (p->flags & TA_FLAG_ASYNC) != 0;
        job.counts = (p->flags & TA_FLAG_DEBUG_COUNTS) != 0;
        job.F = feat_out[t];
        job.A = alpha_out[t];
        job.s = t == 0 ? s : c->aux_stream[t - 1];
        if ((st = raster_pipeline(ct, job)) != TA_OK) {
            if (ct != c) fail(c, st, "target %d: %s", t, ct->err.c_str());
            return st;
        }
    }
    for (int t = 1; t < T; t++) {                         // the call completes on `stream` only
        TA_CUDA(c, cudaEventRecord(c->aux_ev[t], c->aux_stream[t - 1]));
        TA_CUDA(c, cudaStreamWaitEvent(s, c->aux_ev[t], 0));
    }
    return TA_OK;
}

ta_status ta_zbuffer(ta_context* c, const ta_source_view* views, int32_t V, const ta_raster_params* p,
                     const ta_intrinsics* K, const ta_extrinsics* RT, int32_t H, int32_t W, int32_t radius,
                     float baseline_tgt, float* depth_out, float* disp_out, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!views || !p || !K || !RT || !depth_out) return fail(c, TA_ERR_INVALID_ARG, "ta_zbuffer: NULL argument");
    if (V < 1 || V > TA_MAX_VIEWS) return fail(c, TA_ERR_UNSUPPORTED, "ta_zbuffer: V = %d not in [1, %d]", V, TA_MAX_VIEWS);
    if (H < 1 || W < 1 || H > 32767 || W > 32767) return fail(c, TA_ERR_INVALID_ARG, "bad target size %d x %d", H, W);
    if (radius < 0 || radius > 8) return fail(c, TA_ERR_INVALID_ARG, "splat radius %d not in [0, 8]", radius);
    if (disp_out && !(baseline_tgt > 0.0f && std::isfinite(baseline_tgt)))
        return fail(c, TA_ERR_INVALID_ARG, "baseline_tgt must be > 0 when disp_out is given");
    if (!std::isfinite(p->z_near) || !std::isfinite(p->d_min)) return fail(c, TA_ERR_INVALID_ARG, "non-finite params");
    ta_status st;
    if (!finite_cam(*K, *RT, c, &st)) return st;
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    ViewTable vt;
    int64_t pixels = 0;
    uint32_t blocks = 0;
    if ((st = build_view_table(c, views, V, p, false, 8, 4, &vt, &pixels, &blocks)) != TA_OK) return st;
    if (pixels >= (1ll << 32)) return fail(c, TA_ERR_CAPACITY, "more than 2^32 source pixels");
    const uint32_t npix = (uint32_t)H * (uint32_t)W;
    if ((st = grow(c, c->zkey, (size_t)npix * 8)) != TA_OK) return st;
    TargetCam cam;
    cam.fx = K->fx; cam.fy = K->fy; cam.cx = K->cx; cam.cy = K->cy;
    memcpy(cam.R, RT->R, sizeof(cam.R));
    memcpy(cam.t, RT->t, sizeof(cam.t));
    cam.W = W; cam.H = H;
    cam.Wm1f = (float)(W - 1);
    cam.Hm1f = (float)(H - 1);
    unsigned long long* zk = (unsigned long long*)c->zkey.p;
    const unsigned grid = (unsigned)std::min<uint32_t>((npix + 255) / 256, 8u * (uint32_t)c->num_sms);
    k_zb_clear<<<grid, 256, 0, s>>>(zk, npix);
    TA_LAUNCHED(c);
    if (blocks > 0) {
        k_zb_splat<<<blocks, kUnprojThreads, 0, s>>>(vt, cam, p->z_near, radius, zk);
        TA_LAUNCHED(c);
    }
    k_zb_resolve<<<grid, 256, 0, s>>>(zk, npix, K->fx, baseline_tgt, depth_out, disp_out);
    TA_LAUNCHED(c);
    return TA_OK;
}

void ta_default_blend_params(ta_blend_params* bp) {
    if (!bp) return;
    bp->delta = 0.01f;
    bp->edge_tau = 0.02f;
    bp->w_min = 1e-4f;
    bp->tau_c = 0.15f;
}

ta_status ta_blend(ta_context* c, const ta_source_view* views, int32_t V, const float* const* colors,
                   const ta_raster_params* p, const ta_blend_params* bp, const ta_intrinsics* K,
                   const ta_extrinsics* RT, int32_t H, int32_t W, const float* z_fused, float* rgb_out,
                   float* wsum_out, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!views || !colors || !p || !bp || !K || !RT || !z_fused || !rgb_out)
        return fail(c, TA_ERR_INVALID_ARG, "ta_blend: NULL argument");
    if (V < 1 || V > TA_MAX_VIEWS) return fail(c, TA_ERR_UNSUPPORTED, "ta_blend: V = %d not in [1, %d]", V, TA_MAX_VIEWS);
    if (H < 1 || W < 1 || H > 32767 || W > 32767) return fail(c, TA_ERR_INVALID_ARG, "bad target size %d x %d", H, W);
    if (!(bp->delta > 0.0f) || !(bp->edge_tau > 0.0f) || !(bp->w_min >= 0.0f) || !(bp->tau_c >= 0.0f) ||
        !std::isfinite(bp->delta) || !std::isfinite(bp->edge_tau) || !std::isfinite(bp->w_min) || !std::isfinite(bp->tau_c))
        return fail(c, TA_ERR_INVALID_ARG, "blend params: delta > 0, edge_tau > 0, w_min >= 0, tau_c >= 0");
    if (!std::isfinite(p->z_near) || !std::isfinite(p->d_min)) return fail(c, TA_ERR_INVALID_ARG, "non-finite params");
    ta_status st;
    if (!finite_cam(*K, *RT, c, &st)) return st;
    BlendTable bt;
    memset(&bt, 0, sizeof(bt));
    bt.V = V;
    bt.d_min = p->d_min; bt.z_near = p->z_near;
    bt.delta = bp->delta; bt.edge_tau = bp->edge_tau; bt.w_min = bp->w_min; bt.tau_c = bp->tau_c;
    for (int i = 0; i < V; i++) {
        const ta_source_view& s = views[i];
        if (s.H < 1 || s.W < 1 || s.H > 32767 || s.W > 32767)
            return fail(c, TA_ERR_INVALID_ARG, "view %d: bad size %d x %d", i, s.H, s.W);
        if (!s.disparity || !colors[i]) return fail(c, TA_ERR_INVALID_ARG, "view %d: NULL disparity / colour", i);
        if (!(s.baseline > 0.0f) || !std::isfinite(s.baseline))
            return fail(c, TA_ERR_INVALID_ARG, "view %d: baseline must be > 0", i);
        if (!finite_cam(s.K, s.RT, c, &st)) return st;
        BlendView& b = bt.v[i];
        b.disp = s.disparity; b.mask = s.mask; b.color = colors[i];
        b.fx = s.K.fx; b.fy = s.K.fy; b.cx = s.K.cx; b.cy = s.K.cy;
        b.fxB = s.K.fx * s.baseline;            // the oracle's (fx * B), one fp32 product
        memcpy(b.R, s.RT.R, sizeof(b.R));
        memcpy(b.t, s.RT.t, sizeof(b.t));
        b.H = s.H; b.W = s.W;
    }
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    TargetCam cam;
    cam.fx = K->fx; cam.fy = K->fy; cam.cx = K->cx; cam.cy = K->cy;
    memcpy(cam.R, RT->R, sizeof(cam.R));
    memcpy(cam.t, RT->t, sizeof(cam.t));
    cam.W = W; cam.H = H;
    cam.Wm1f = (float)(W - 1);
    cam.Hm1f = (float)(H - 1);
    const uint32_t npix = (uint32_t)H * (uint32_t)W;
    k_blend<<<(npix + 255) / 256, 256, 0, s>>>(bt, cam, z_fused, rgb_out, wsum_out);
    TA_LAUNCHED(c);
    return TA_OK;
}

ta_status ta_rasterize_backward(ta_context* c, const ta_gaussians* g, int64_t n, int32_t H, int32_t W,
                                const ta_raster_params* p, const float* grad_F, const float* grad_A, float* d_mean2,
                                float* d_conic, float* d_alpha, float* d_feat, void* stream) {
    if (!c) return TA_ERR_INVALID_ARG;
    if (!g || !p || !grad_F || !grad_A || !d_mean2 || !d_conic || !d_alpha || !d_feat)
        return fail(c, TA_ERR_INVALID_ARG, "ta_rasterize_backward: NULL argument");
    if (!c->have_last || c->last_H != H || c->last_W != W)
        return fail(c, TA_ERR_INVALID_ARG, "ta_rasterize_backward needs the matching ta_rasterize on this context first");
    if (!supported_C(g->C)) return fail(c, TA_ERR_UNSUPPORTED, "C = %d not in {8,16,32,64}", g->C);
    if (n < -1 || (n == -1 && !g->n_dev) || n > g->capacity) return fail(c, TA_ERR_INVALID_ARG, "bad n");
    RasterConsts rc;
    rc.dilation = p->dilation; rc.alpha_max = p->alpha_max; rc.alpha_min = p->alpha_min; rc.t_eps = p->t_eps;
    rc.cull_sigma = p->cull_sigma; rc.z_near = p->z_near;
    rc.q_max = p->cull_sigma * p->cull_sigma;
    rc.q_lo_half = -0.5f * rc.q_max;
    rc.a_max_2k = 2048.0f * p->alpha_max;
    rc.a_min_2k = 2048.0f * p->alpha_min;
    // the pass reuses the forward call's records and tile lists: it must be the same Gaussian set,
    // feature layout, count and constants (a different C would index the feature rows with the wrong
    // stride); grad_F is read with 16-byte vector loads
    const int fbytes = g->feat_dtype == TA_F16 ? 2 : 4;
    if (g->C != c->last_C || fbytes != c->last_fbytes || n != c->last_n || g->feat != c->last_feat ||
        memcmp(&rc, &c->last_rc, sizeof(rc)) != 0)
        return fail(c, TA_ERR_INVALID_ARG, "ta_rasterize_backward: C, feature dtype/array, n or params differ from the "
                                           "preceding ta_rasterize on this context");
    if ((((uintptr_t)grad_F) | ((uintptr_t)d_feat)) & 15)
        return fail(c, TA_ERR_INVALID_ARG, "grad_F / d_feat must be 16-byte aligned");
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const CompositeGeom& cg = c->last_cg;
    cudaError_t e = launch_composite_bwd(g->C, fbytes, cg.TX * cg.TY, c->resident_bwd, c->bwd_simt, (const uint4*)c->last_rec,
                                         g->feat, (const uint32_t*)c->tlist.p, (const uint2*)c->trng.p,
                                         (const uint32_t*)c->tile_order.p, cg, rc,
                                         (CallState*)c->cs.p, (uint64_t)(c->tlist.bytes / 4), grad_F, grad_A,
                                         d_mean2, d_conic, d_alpha, d_feat, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "backward launch");
    c->launches += 2;   // k_bwd_zero + k_composite_bwd
    return TA_OK;
}

ta_status ta_debug_last(ta_context* c, ta_debug_view* out, void* stream) {
    if (!c || !out) return TA_ERR_INVALID_ARG;
    if (!c->have_last) return fail(c, TA_ERR_INVALID_ARG, "no rasterize call yet");
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    CallState* cs = (CallState*)c->cs.p;
    const CompositeGeom& cg = c->last_cg;
    const int T = cg.TX * cg.TY;
    ta_status st;
    if ((st = grow(c, c->dbg_offs, ((size_t)T + 1) * 4 + 64)) != TA_OK) return st;
    unsigned long long* status = (unsigned long long*)c->status.p + (size_t)5 * c->status_region;
    if (scan_tiles((uint32_t)T + 1) > c->status_region) return fail(c, TA_ERR_CAPACITY, "debug scan status too small");
    TA_CUDA(c, cudaMemsetAsync(status, 0, (size_t)c->status_region * 8, s));
    TA_CUDA(c, cudaMemsetAsync(&cs->scan_counter[5], 0, 4, s));
    launch_debug_tile_lists((const uint2*)c->trng.p, (const uint32_t*)c->tlist.p, cg, (uint32_t*)c->dbg_offs.p, status,
                            &cs->scan_counter[5], &cs->sort_total, nullptr, 0, 0, s);
    TA_CUDA(c, cudaGetLastError());
    CallState h;
    TA_CUDA(c, cudaMemcpyAsync(&h, c->cs.p, sizeof(CallState), cudaMemcpyDeviceToHost, s));
    TA_CUDA(c, cudaStreamSynchronize(s));
    const uint64_t K = h.sort_total;
    if ((st = grow(c, c->dbg_list, (size_t)std::max<uint64_t>(K, 1) * 4)) != TA_OK) return st;
    launch_debug_tile_lists((const uint2*)c->trng.p, (const uint32_t*)c->tlist.p, cg, (uint32_t*)c->dbg_offs.p, status,
                            &cs->scan_counter[5], &cs->sort_total, (uint32_t*)c->dbg_list.p, K, 1, s);
    TA_CUDA(c, cudaGetLastError());
    TA_CUDA(c, cudaStreamSynchronize(s));
    int passes = 0;
    const uint32_t m = h.key_or ^ h.key_and;
    if (h.n_visible && m) {
        int lo = 0, hi = 31;
        while (!((m >> lo) & 1u)) lo++;
        while (!((m >> hi) & 1u)) hi--;
        passes = (hi - lo) / 8 + 1;
    }
    out->n = h.n;
    out->K = (int64_t)K;
    out->Kc = (int64_t)h.K;
    out->P = (int32_t)h.bin_P;
    out->tiles_x = cg.TX;
    out->tiles_y = cg.TY;
    out->sort_passes = passes;
    out->records = (const uint32_t*)c->last_rec;
    out->depth_keys = (const uint32_t*)c->last_k[passes & 1];
    out->order = (const uint32_t*)c->last_v[passes & 1];
    out->tile_offsets = (const uint32_t*)c->dbg_offs.p;
    out->tile_list = (const uint32_t*)c->dbg_list.p;
    out->n_contrib = c->last_counts ? (const int32_t*)c->ncontrib.p : nullptr;
    for (int k = 0; k < 8; k++) out->work[k] = c->last_counts ? (int64_t)h.work[k] : 0;
    out->tile_px = 1 << cg.ts;
    out->reserved = 0;
    return TA_OK;
}

ta_status ta_profile_enable(ta_context* c, int32_t enable) {
    if (!c) return TA_ERR_INVALID_ARG;
    c->profiling = enable != 0;
    return TA_OK;
}

ta_status ta_profile_read(ta_context* c, ta_profile* out, int32_t reset) {
    if (!c) return TA_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    TA_CUDA(c, cudaDeviceSynchronize());
    for (auto& p : c->pending) {
        float ms = 0.0f;
        TA_CUDA(c, cudaEventElapsedTime(&ms, p.a, p.b));
        c->prof_ms[p.stage] += ms;
        c->prof_calls[p.stage] += 1;
        c->pool.push_back(p);
    }
    c->pending.clear();
    if (out) {
        for (int i = 0; i < TA_STAGE_COUNT; i++) { out->ms[i] = c->prof_ms[i]; out->calls[i] = c->prof_calls[i]; }
    }
    if (reset) {
        for (int i = 0; i < TA_STAGE_COUNT; i++) { c->prof_ms[i] = 0.0; c->prof_calls[i] = 0; }
    }
    return TA_OK;
}

ta_status ta_check_overflow(ta_context* c, void* stream, int32_t* overflowed) {
    if (!c) return TA_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    CallState h;
    TA_CUDA(c, cudaMemcpyAsync(&h, c->cs.p, sizeof(CallState), cudaMemcpyDeviceToHost, s));
    TA_CUDA(c, cudaStreamSynchronize(s));
    const uint32_t zero = 0;
    TA_CUDA(c, cudaMemcpy((char*)c->cs.p + offsetof(CallState, overflow), &zero, 4, cudaMemcpyHostToDevice));
    bool over = h.overflow != 0;
    for (int k = 0; k < kMaxFrontTargets - 1; k++) {        // the lanes' child contexts
        if (!c->aux[k]) continue;
        TA_CUDA(c, cudaStreamSynchronize(c->aux_stream[k]));
        int32_t o = 0;
        ta_check_overflow(c->aux[k], (void*)c->aux_stream[k], &o);
        over = over || o != 0;
    }
    if (overflowed) *overflowed = over ? 1 : 0;
    return over ? fail(c, TA_ERR_CAPACITY, "tile-entry capacity overflowed in an async call") : TA_OK;
}

}  // extern "C"
