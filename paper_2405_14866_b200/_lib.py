"""ctypes binding of include/ta.h -- argument marshalling only.

Every step of the hot path runs in libtaloha.so (CUDA, sm_100a).  There is no CPU fallback:
if the shared library is missing or no CUDA device is present, these calls raise.
Tensors are torch CUDA tensors (PyTorch supplies device memory and streams only).
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

TA_F32, TA_F16 = 0, 1
TA_FLAG_ASYNC, TA_FLAG_DEBUG_COUNTS = 1, 2
TA_MAX_VIEWS = 16
STATUS = {0: "TA_OK", 1: "TA_ERR_INVALID_ARG", 2: "TA_ERR_UNSUPPORTED", 3: "TA_ERR_CUDA",
          4: "TA_ERR_OUT_OF_MEMORY", 5: "TA_ERR_CAPACITY"}


class TaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float)]


class Extrinsics(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3)]


class SourceView(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("disparity", C.c_void_p), ("mask", C.c_void_p),
                ("K", Intrinsics), ("RT", Extrinsics), ("baseline", C.c_float), ("scale", C.c_void_p),
                ("quat", C.c_void_p), ("opacity", C.c_void_p), ("feat", C.c_void_p)]


class Gaussians(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("n_dev", C.c_void_p), ("pos_alpha", C.c_void_p), ("cov", C.c_void_p),
                ("feat", C.c_void_p), ("C", C.c_int32), ("feat_dtype", C.c_int32)]


class RasterParams(C.Structure):
    _fields_ = [("dilation", C.c_float), ("alpha_max", C.c_float), ("alpha_min", C.c_float),
                ("t_eps", C.c_float), ("cull_sigma", C.c_float), ("z_near", C.c_float), ("d_min", C.c_float),
                ("default_scale", C.c_float), ("default_opacity", C.c_float), ("flags", C.c_uint32),
                ("exact_exp", C.c_int32)]


class BlendParams(C.Structure):
    _fields_ = [("delta", C.c_float), ("edge_tau", C.c_float), ("w_min", C.c_float), ("tau_c", C.c_float)]


class DebugView(C.Structure):
    _fields_ = [("n", C.c_int64), ("K", C.c_int64), ("Kc", C.c_int64), ("P", C.c_int32), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32), ("sort_passes", C.c_int32), ("records", C.c_void_p),
                ("depth_keys", C.c_void_p), ("order", C.c_void_p), ("tile_offsets", C.c_void_p),
                ("tile_list", C.c_void_p), ("n_contrib", C.c_void_p),
                ("work", C.c_int64 * 8), ("tile_px", C.c_int32), ("reserved", C.c_int32)]


STAGES = ("unproject", "project", "sort", "bin_count", "bin_scan", "bin_place", "composite")


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("calls", C.c_uint64 * 7)]


EXPORTS = ("ta_rasterize_views", "ta_render_sources", "ta_profile_enable", "ta_profile_read", "ta_default_params", "ta_context_create", "ta_context_destroy", "ta_reserve", "ta_unproject",
           "ta_zbuffer", "ta_blend", "ta_default_blend_params", "ta_rasterize_backward",
           "ta_rasterize", "ta_debug_last", "ta_check_overflow", "ta_launch_count", "ta_status_string",
           "ta_last_error", "ta_build_info")

_lib = None


def lib(build_if_stale: bool = False):
    """Load libtaloha.so (in-tree).  Raises if it is missing: the product path has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_stale and _build.stale():
        _build.build()
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"{_build.LIB} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(_build.LIB)
    P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.ta_default_params.argtypes = [C.POINTER(RasterParams)]
    L.ta_default_params.restype = None
    L.ta_context_create.argtypes = [i32, C.POINTER(P)]
    L.ta_context_destroy.argtypes = [P]
    L.ta_reserve.argtypes = [P, i64, i64, i32, i32]
    L.ta_unproject.argtypes = [P, C.POINTER(SourceView), i32, C.POINTER(RasterParams), C.POINTER(Gaussians), P]
    L.ta_rasterize.argtypes = [P, C.POINTER(Gaussians), i64, C.POINTER(Intrinsics), C.POINTER(Extrinsics), i32, i32,
                               C.POINTER(RasterParams), P, P, P]
    L.ta_debug_last.argtypes = [P, C.POINTER(DebugView), P]
    L.ta_default_blend_params.argtypes = [C.POINTER(BlendParams)]
    L.ta_rasterize_backward.argtypes = [P, C.POINTER(Gaussians), i64, i32, i32, C.POINTER(RasterParams), P, P, P, P, P,
                                        P, P]
    L.ta_blend.argtypes = [P, C.POINTER(SourceView), i32, C.POINTER(P), C.POINTER(RasterParams), C.POINTER(BlendParams),
                           C.POINTER(Intrinsics), C.POINTER(Extrinsics), i32, i32, P, P, P, P]
    L.ta_zbuffer.argtypes = [P, C.POINTER(SourceView), i32, C.POINTER(RasterParams), C.POINTER(Intrinsics),
                             C.POINTER(Extrinsics), i32, i32, i32, C.c_float, P, P, P]
    L.ta_check_overflow.argtypes = [P, P, C.POINTER(i32)]
    L.ta_rasterize_views.argtypes = [P, C.POINTER(Gaussians), i64, i32, C.POINTER(Intrinsics), C.POINTER(Extrinsics),
                                     i32, i32, C.POINTER(RasterParams), C.POINTER(P), C.POINTER(P), i32, P]
    L.ta_render_sources.argtypes = [P, C.POINTER(SourceView), i32, i32, i32, C.POINTER(RasterParams), i32,
                                    C.POINTER(Intrinsics), C.POINTER(Extrinsics), i32, i32, C.POINTER(P), C.POINTER(P), P]
    L.ta_profile_enable.argtypes = [P, i32]
    L.ta_profile_read.argtypes = [P, C.POINTER(Profile), i32]
    L.ta_launch_count.argtypes = [P]
    L.ta_launch_count.restype = C.c_uint64
    L.ta_status_string.argtypes = [i32]
    L.ta_status_string.restype = C.c_char_p
    L.ta_last_error.argtypes = [P]
    L.ta_last_error.restype = C.c_char_p
    L.ta_build_info.restype = C.c_char_p
    for name in ("ta_context_create", "ta_context_destroy", "ta_reserve", "ta_unproject", "ta_rasterize", "ta_zbuffer",
                 "ta_blend", "ta_rasterize_backward", "ta_render_sources", "ta_rasterize_views",
                 "ta_debug_last", "ta_check_overflow", "ta_profile_enable", "ta_profile_read"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def default_params(**kw) -> RasterParams:
    p = RasterParams()
    lib().ta_default_params(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def intrinsics(K) -> Intrinsics:
    return Intrinsics(*[float(v) for v in K])


def extrinsics(R, t) -> Extrinsics:
    e = Extrinsics()
    for i, v in enumerate(list(R)):
        e.R[i] = float(v)
    for i, v in enumerate(list(t)):
        e.t[i] = float(v)
    return e


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _raw(t):
    """A device address: a CUDA tensor's data pointer, or an integer address as is (e.g. a peer mapping
    opened with CUDA IPC, paper_2405_14866_b200.dist.PeerFrame)."""
    return int(t) if isinstance(t, int) else t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class Context:
    """A ta_context on one CUDA device (owns grow-only scratch)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        st = lib().ta_context_create(int(device), C.byref(self._h))
        if st != 0:
            raise TaError(st, "ta_context_create failed (is a CUDA device present?)")
        self.device = device

    def _check(self, st):
        if st != 0:
            raise TaError(st, lib().ta_last_error(self._h).decode())

    def close(self):
        if self._h:
            lib().ta_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().ta_launch_count(self._h))

    def reserve(self, max_gaussians, max_entries, H, W):
        self._check(lib().ta_reserve(self._h, int(max_gaussians), int(max_entries), int(H), int(W)))

    def unproject(self, views, params: RasterParams, g: "GaussianBuffers", stream=None):
        arr = (SourceView * len(views))(*views)
        gs = g.struct()
        self._check(lib().ta_unproject(self._h, arr, len(views), C.byref(params), C.byref(gs), _stream(stream)))

    def zbuffer(self, views, params: RasterParams, K: Intrinsics, RT: Extrinsics, H, W, radius, baseline_tgt,
                depth_out, disp_out=None, stream=None):
        """NEXT #2 cascade Z-buffer (include/ta.h ta_zbuffer): views = SourceView structs."""
        arr = (SourceView * len(views))(*views)
        self._check(lib().ta_zbuffer(self._h, arr, len(views), C.byref(params), C.byref(K), C.byref(RT), int(H),
                                     int(W), int(radius), float(baseline_tgt), _ptr(depth_out), _ptr(disp_out),
                                     _stream(stream)))

    def blend(self, views, colors, params: RasterParams, bp: "BlendParams", K: Intrinsics, RT: Extrinsics, H, W,
              z_fused, rgb_out, wsum_out=None, stream=None):
        """NEXT #1 occlusion-aware blending (include/ta.h ta_blend): colors = CUDA tensors [H_i, W_i, 3]."""
        arr = (SourceView * len(views))(*views)
        cp = (C.c_void_p * len(colors))(*[c.data_ptr() for c in colors])
        self._check(lib().ta_blend(self._h, arr, len(views), cp, C.byref(params), C.byref(bp), C.byref(K), C.byref(RT),
                                   int(H), int(W), _ptr(z_fused), _ptr(rgb_out), _ptr(wsum_out), _stream(stream)))

    def rasterize_backward(self, g: "GaussianBuffers", n, H, W, params: RasterParams, grad_F, grad_A, d_mean2, d_conic,
                           d_alpha, d_feat, stream=None):
        """NEXT #4 (include/ta.h ta_rasterize_backward): after ta_rasterize of the same inputs."""
        gs = g.struct()
        self._check(lib().ta_rasterize_backward(self._h, C.byref(gs), int(n), int(H), int(W), C.byref(params),
                                                _ptr(grad_F), _ptr(grad_A), _ptr(d_mean2), _ptr(d_conic),
                                                _ptr(d_alpha), _ptr(d_feat), _stream(stream)))

    def rasterize(self, g: "GaussianBuffers", n, K: Intrinsics, RT: Extrinsics, H, W, params: RasterParams,
                  feat_out, alpha_out, stream=None):
        gs = g.struct()
        self._check(lib().ta_rasterize(self._h, C.byref(gs), int(n), C.byref(K), C.byref(RT), int(H), int(W),
                                       C.byref(params), _ptr(feat_out), _ptr(alpha_out), _stream(stream)))

    def rasterize_views(self, g: "GaussianBuffers", n, Ks, RTs, H, W, params: RasterParams, feat_outs, alpha_outs,
                        lanes: int = 4, stream=None):
        """Multi-view rendering (include/ta.h ta_rasterize_views): one Gaussian set into len(Ks) targets,
        spread over `lanes` (context, stream) lanes inside the library; Ks / RTs = Intrinsics / Extrinsics
        structs, feat_outs / alpha_outs = CUDA tensors [H, W, C] / [H, W] per target or integer device addresses
        (e.g. views of another rank's frame buffer mapped over NVLink, dist.PeerFrame)."""
        T = len(Ks)
        gs = g.struct()
        ka = (Intrinsics * T)(*Ks)
        ra = (Extrinsics * T)(*RTs)
        fo = (C.c_void_p * T)(*[_raw(f) for f in feat_outs])
        ao = (C.c_void_p * T)(*[_raw(a) for a in alpha_outs])
        self._check(lib().ta_rasterize_views(self._h, C.byref(gs), int(n), T, ka, ra, int(H), int(W), C.byref(params),
                                             fo, ao, int(lanes), _stream(stream)))

    def render_sources(self, views, C_: int, feat_dtype: str, params: RasterParams, Ks, RTs, H, W, feat_outs, alpha_outs,
                       stream=None):
        """north_star (a) fused front end (include/ta.h ta_render_sources): lift + project + cull straight from
        the source views for len(Ks) targets, then bin / sort / composite each; Ks / RTs = Intrinsics /
        Extrinsics structs, feat_outs / alpha_outs = CUDA tensors [H, W, C] / [H, W] per target."""
        T = len(Ks)
        arr = (SourceView * len(views))(*views)
        ka = (Intrinsics * T)(*Ks)
        ra = (Extrinsics * T)(*RTs)
        fo = (C.c_void_p * T)(*[f.data_ptr() for f in feat_outs])
        ao = (C.c_void_p * T)(*[a.data_ptr() for a in alpha_outs])
        self._check(lib().ta_render_sources(self._h, arr, len(views), int(C_), TA_F16 if feat_dtype == "f16" else TA_F32,
                                            C.byref(params), T, ka, ra, int(H), int(W), fo, ao, _stream(stream)))

    def profile(self, enable: bool):
        self._check(lib().ta_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self, reset: bool = True) -> dict:
        """Per-stage {name: (total_ms, calls)} of the event pairs recorded since the last reset."""
        p = Profile()
        self._check(lib().ta_profile_read(self._h, C.byref(p), 1 if reset else 0))
        return {name: (p.ms[i], int(p.calls[i])) for i, name in enumerate(STAGES)}

    def debug_last(self, stream=None) -> DebugView:
        d = DebugView()
        self._check(lib().ta_debug_last(self._h, C.byref(d), _stream(stream)))
        return d

    def check_overflow(self, stream=None) -> bool:
        o = C.c_int32(0)
        st = lib().ta_check_overflow(self._h, _stream(stream), C.byref(o))
        if st not in (0, 5):
            self._check(st)
        return bool(o.value)


class GaussianBuffers:
    """Device SoA of a Gaussian set (include/ta.h ta_gaussians) held in torch CUDA tensors."""

    def __init__(self, capacity: int, C_: int, feat_dtype: str, device="cuda"):
        import torch
        self.capacity = int(capacity)
        self.C = int(C_)
        self.feat_dtype = feat_dtype
        cap = max(1, self.capacity)
        self.pos_alpha = torch.empty((cap, 4), dtype=torch.float32, device=device)
        self.cov = torch.empty((cap, 8), dtype=torch.float32, device=device)
        self.feat = torch.empty((cap, self.C), dtype=torch.float16 if feat_dtype == "f16" else torch.float32,
                                device=device)
        self.n_dev = torch.zeros(1, dtype=torch.int64, device=device)

    def struct(self) -> Gaussians:
        return Gaussians(self.capacity, _ptr(self.n_dev), _ptr(self.pos_alpha), _ptr(self.cov), _ptr(self.feat),
                         self.C, TA_F16 if self.feat_dtype == "f16" else TA_F32)

    @property
    def n(self) -> int:
        return int(self.n_dev.item())


def source_view(H, W, disparity, mask, K, R, t, baseline, scale, quat, opacity, feat) -> SourceView:
    """Marshal one source view of device tensors (None -> NULL) into the C struct."""
    return SourceView(int(H), int(W), _ptr(disparity), _ptr(mask), intrinsics(K), extrinsics(R, t), float(baseline),
                      _ptr(scale), _ptr(quat), _ptr(opacity), _ptr(feat))


def default_blend_params(**kw) -> BlendParams:
    bp = BlendParams()
    lib().ta_default_blend_params(C.byref(bp))
    for k, v in kw.items():
        setattr(bp, k, v)
    return bp
