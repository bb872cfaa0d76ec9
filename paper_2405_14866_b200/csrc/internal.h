// internal.h -- kernel parameter structs and kernel declarations shared by the .cu files.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace ta {

struct TargetCam {
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    int W, H;
    float Wm1f, Hm1f;     // (float)(W-1), (float)(H-1): exact for W, H < 2^24
};

struct RasterConsts {
    float dilation, alpha_max, alpha_min, t_eps, cull_sigma, z_near, q_max;
    // the compositors' staged scalings (exact powers of two): -q_max / 2, 2^11 alpha_max, 2^11 alpha_min
    // -- kernel parameters, so the per-entry compares and clamps read them as constant operands
    float q_lo_half, a_max_2k, a_min_2k;
};

struct BinGeom {
    int shift;            // bin = (1 << shift) x (1 << shift) pixels (coarse bins: 32 x 32)
    int ts;               // compositing tile = (1 << ts) x (1 << ts) pixels (3 or 4); shift - ts = 1 or 2
    int TX, TY;           // bins per row / column
    int nw;               // warps per k_bin_place block (per-warp [NB] cursors in shared memory)
    uint32_t P;           // rank tiles = columns of the bin-major [NB x P] run-start matrix
};

struct ViewDesc {
    const float* disp;
    const uint8_t* mask;
    const float* scale;
    const float* quat;
    const float* opacity;
    const void* feat;
    float fx, fy, cx, cy;
    float R[9];
    float t[3];
    float baseline;
    int H, W;
    uint32_t blk_begin;   // first unprojection block of this view
    uint32_t idx0;        // running pixel offset of this view (z-buffer source index)
    int vec4;             // 1: H*W % 4 == 0 and all maps 16-byte aligned -> 128-bit loads
};

constexpr int kMaxViews = 16;
struct ViewTable {
    ViewDesc v[kMaxViews];
    int V;
    int C;
    int fbytes;           // 2 (f16) or 4 (f32)
    float d_min, default_scale, default_opacity;
};

constexpr int kUnprojThreads = 256;
constexpr int kUnprojPix = 4 * kUnprojThreads;   // pixels per block

// raster.cu
__global__ void k_init(CallState* cs, unsigned long long* status, int n_status, int64_t n_host,
                       const int64_t* n_dev, uint32_t bin_ranks, uint32_t nbins, const uint32_t* stats);
__global__ void k_project(const float4* pos_alpha, const float4* cov, TargetCam cam, RasterConsts rc,
                          CallState* cs, uint4* rec, uint32_t* key0, uint32_t* val0);
__global__ void k_sort_digits(const uint32_t* keys, CallState* cs);
__global__ void k_sort_pass(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b, int pass,
                            CallState* cs, unsigned long long* lb, const uint4* rec, uint2* boxes);
__global__ void k_gather_boxes(const uint4* rec, const uint32_t* vals_a, const uint32_t* vals_b, const CallState* cs,
                               uint2* boxes);
__global__ void k_bin_count(const uint2* boxes, const CallState* cs, BinGeom bg, uint32_t* counts);
__global__ void k_bin_place(const uint2* boxes, const uint32_t* vals_a, const uint32_t* vals_b, CallState* cs,
                            BinGeom bg, const uint32_t* offs, uint32_t* list, uint64_t list_cap);
constexpr uint32_t kBinTileRanks(int nw) { return (uint32_t)nw * 256u; }

// In-place exclusive scan of data[0 .. len) with len = *len_ptr (device) or len_max (len_ptr NULL);
// status (>= len_max/4096 + 1 words) and *counter must be zero.
void launch_scan(uint32_t* data, const uint32_t* len_ptr, uint32_t len_max, unsigned long long* status,
                 uint32_t* counter, unsigned long long* total, cudaStream_t st);
constexpr uint32_t scan_tiles(uint32_t len_max) { return len_max / 4096u + 1u; }

// composite.cu
struct CompositeGeom {
    int TX, TY;           // compositing tiles ((1 << ts) pixels square) per row / column
    int W, H;
    int shift, BX;        // coarse bins: (1 << shift) pixels square, BX per row
    int ts;               // tile side 1 << ts: 8 (one warp block per tile) or 16 (four 8 x 8 blocks)
    uint32_t P;           // coarse-binning partitions (columns of the bin-major offset matrix)
};
// per-tile lists (tile, depth, id) from the coarse bin lists: tlist + trng[tile] = (start, count)
void launch_tile_split(const uint32_t* clist, const uint32_t* coffs, CompositeGeom cg,
                       const CallState* cs, uint64_t clist_cap, uint32_t* tlist, uint64_t tlist_cap, uint2* trng,
                       cudaStream_t st);
// per-device preparation (ta_context_create): shared-memory opt-ins + persistent grid sizes per C
// (slot c_slot(C): C = 8, 16, 32, 64; slots 4 / 5: the tensor-memory-accumulator variant, C = 32 / 64)
cudaError_t prepare_composite(int num_sms, int ctas_per_sm_cap, int resident[6]);
int c_slot(int C);
cudaError_t launch_composite(int C, int fbytes, int tiles, const int* resident, bool fast_exp, const uint4* rec, const void* feat,
                             const uint32_t* tlist, const uint2* trng, uint32_t* order, CompositeGeom cg,
                             RasterConsts rc, const CallState* cs, uint64_t list_cap, float* F, float* A,
                             int32_t* ncontrib, cudaStream_t st, bool tm_acc = false);
// heaviest-first tile order (by list length) for the persistent compositors
void launch_tile_order(const uint2* trng, CompositeGeom cg, uint32_t* order, cudaStream_t st);
// composite_tm.cu: tensor-memory compositor (fp16 features, C in {16, 32, 64}); resident[c_slot(C)]
cudaError_t prepare_composite_tm(int num_sms, int ctas_per_sm_cap, int resident[4]);
cudaError_t launch_composite_tm(int C, int tiles, const int* resident, bool fast_exp, const uint4* rec, const void* feat,
                                const uint32_t* tlist, const uint2* trng, const uint32_t* order, CompositeGeom cg,
                                RasterConsts rc, const CallState* cs, uint64_t list_cap, float* F, float* A,
                                int32_t* ncontrib, cudaStream_t st);
// composite_ws.cu: warp-specialized compositor (producer / consumer warp pairs; fp16 C = 32, 16 x 16 tiles)
// (resident[0]: 1 producer : 1 consumer, resident[1]: 1 : 2)
cudaError_t prepare_composite_ws(int num_sms, int cap, int* resident);
cudaError_t launch_composite_ws(int cpp, int tiles, const int* resident, bool fast, const uint4* rec, const void* feat,
                                const uint32_t* list, const uint2* trng, uint32_t* order, CompositeGeom cg, RasterConsts rc,
                                const CallState* cs, uint64_t list_cap, float* F, float* A, int32_t* ncontrib,
                                cudaStream_t st);
// backward.cu
cudaError_t prepare_composite_bwd(int num_sms, int resident[4]);
cudaError_t launch_composite_bwd(int C, int fbytes, int tiles, const int* resident, bool simt, const uint4* rec, const void* feat, const uint32_t* tlist,
                                 const uint2* trng, const uint32_t* order, CompositeGeom cg, RasterConsts rc,
                                 CallState* cs, uint64_t list_cap, const float* GF, const float* GA, float* d_mean2,
                                 float* d_conic, float* d_alpha, float* d_feat, cudaStream_t st);
// debug: compact the per-tile (tile, depth, id) lists the compositor walks into one array (a3/a5 check)
void launch_debug_tile_lists(const uint2* trng, const uint32_t* tlist, CompositeGeom cg, uint32_t* tile_offs,
                             unsigned long long* status, uint32_t* counter, unsigned long long* total, uint32_t* out_list,
                             uint64_t out_cap, int pass, cudaStream_t st);

// blend.cu
struct BlendView {
    const float* disp;
    const uint8_t* mask;
    const float* color;   // [H][W][3]
    float fx, fy, cx, cy, fxB;
    float R[9], t[3];
    int H, W;
};
struct BlendTable {
    BlendView v[kMaxViews];
    int V;
    float d_min, z_near, delta, edge_tau, w_min, tau_c;
};
__global__ void k_blend(BlendTable bt, TargetCam cam, const float* zf, float* rgb, float* wsum);

// zbuffer.cu
__global__ void k_zb_clear(unsigned long long* zk, uint32_t n);
__global__ void k_zb_splat(ViewTable vt, TargetCam cam, float z_near, int radius, unsigned long long* zk);
__global__ void k_zb_resolve(const unsigned long long* zk, uint32_t n, float fx, float baseline, float* depth,
                             float* disp);

// unproject.cu
__global__ void k_unproject_count(ViewTable vt, uint32_t* counts);
// fused front end (north_star (a)): up to kMaxFrontTargets targets per call
constexpr int kMaxFrontTargets = 4;
struct FrontTargets {
    TargetCam cam[kMaxFrontTargets];
    uint4* rec[kMaxFrontTargets];
    uint32_t* key[kMaxFrontTargets];
    uint32_t* val[kMaxFrontTargets];
    int T;
};
__global__ void k_front_fused(ViewTable vt, const uint32_t* offs, FrontTargets ft, RasterConsts rc, void* feat_out,
                              uint32_t* stats);
__global__ void k_front_stats_init(uint32_t* stats, int T);
__global__ void k_unproject_write(ViewTable vt, const uint32_t* offs, float4* pos_alpha, float4* cov, void* feat);

}  // namespace ta
