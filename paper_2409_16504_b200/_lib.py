"""ctypes binding of libsfb200.so (the C ABI declared in include/sfb200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every entry point raises. Device buffers come from torch
(``tensor.data_ptr()``); launches go on torch's current CUDA stream so torch
events and the library's kernels share one timeline.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SFB_LIB_PATH", PKG / "_build" / "libsfb200.so"))   # env: A/B builds

SFB_OK, SFB_ERR_ARG, SFB_ERR_OOM, SFB_ERR_CUDA, SFB_ERR_STATE = 0, 1, 2, 3, 4
PLANE_RGB, PLANE_NORMAL, PLANE_DEPTH = 1, 2, 4
NET_SIMT_F32, NET_TC_TF32X3, NET_TC_BF16, NET_SIMT_F64 = 0, 1, 2, 3
STAGES = {1: "voxelize", 2: "unet", 3: "head", 4: "project", 5: "sort", 6: "bin",
          7: "composite", 8: "composite_reps", 9: "untimed"}
COMPOSITE_REPS = 4   # render.cu kCompReps: back-to-back compositor launches in stage timing

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double


class Camera_t(ctypes.Structure):
    _fields_ = [("rot", D * 9), ("trans", D * 3), ("fx", D), ("fy", D), ("cx", D), ("cy", D),
                ("width", I32), ("height", I32)]


class RenderOptions_t(ctypes.Structure):
    _fields_ = [("tile_size", I32), ("early_termination", I32), ("alpha_max", D)]


class Splats_t(ctypes.Structure):
    _fields_ = [("centers", P), ("scales", P), ("quaternions", P), ("opacities", P),
                ("colors", P), ("normals", P), ("n", I64)]


class Shading_t(ctypes.Structure):
    _fields_ = [("mode", I32), ("light", D * 3), ("ambient", D), ("diffuse", D)]


class Stats_t(ctypes.Structure):
    _fields_ = [("kept", I64), ("runs", I64), ("fine_entries", I64), ("super_entries", I64),
                ("global_entries", I64), ("voxels", I64 * 8)]


# name -> argtypes (restype is always int)
SIGNATURES = {
    "sfb_ctx_create": [ctypes.c_int, ctypes.POINTER(P)],
    "sfb_ctx_destroy": [P],
    "sfb_last_error": [P],
    "sfb_set_stream": [P, P],
    "sfb_get_stats": [P, ctypes.POINTER(Stats_t)],
    "sfb_version": [],
    "sfb_set_timing": [P, ctypes.c_int],
    "sfb_set_graphs": [P, ctypes.c_int],
    "sfb_set_entry_capacity": [P, I64],
    "sfb_set_conv_staging": [P, ctypes.c_int],
    "sfb_set_debug_counters": [P, P],
    "sfb_stage_times": [P, P, P, I32, ctypes.POINTER(I32)],
    "sfb_set_frame_debug": [P, I64, P, P, P, P, I32, P, P],
    "sfb_bbox": [P, P, I64, P],
    "sfb_bbox_async": [P, P, I64, P],
    "sfb_voxelize": [P, P, P, I64, D, P, P, P, P, P, P, P, ctypes.POINTER(I64)],
    "sfb_kernel_map": [P, P, I64, I32, I32, P],
    "sfb_transposed_map": [P, P, I64, I32, P, I64, P, P],
    "sfb_pool": [P, P, P, I64, I32, I32, P, P, P, ctypes.POINTER(I64)],
    "sfb_pool_f64": [P, P, P, I64, I32, I32, P, P, P, ctypes.POINTER(I64)],
    "sfb_lookup": [P, P, I64, P, I64, P],
    "sfb_net_load": [P, P, ctypes.c_size_t],
    "sfb_net_set_mode": [P, ctypes.c_int],
    "sfb_layer_set": [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P],
    "sfb_sparse_conv": [P, ctypes.c_int, P, P, I64, I32, ctypes.c_int, P],
    "sfb_transposed_conv": [P, ctypes.c_int, P, P, I64, I32, P, I64, ctypes.c_int, P],
    "sfb_unet_forward": [P, P, P, I64, P],
    "sfb_activate_head": [P, P, I64, D, P, P, P, P, P],
    "sfb_estimate_neural": [P, P, P, I64, D, P, P, P, P, P, P, P],
    "sfb_render": [P, ctypes.POINTER(Splats_t), ctypes.POINTER(Camera_t),
                   ctypes.POINTER(RenderOptions_t), I32, P, P, P, P, P],
    "sfb_project": [P, ctypes.POINTER(Splats_t), ctypes.POINTER(Camera_t), D, D] + [P] * 8,
    "sfb_prepare_debug": [P, ctypes.POINTER(Splats_t), ctypes.POINTER(Camera_t), I32, P, P, P, P,
                          I64, ctypes.POINTER(I64), ctypes.POINTER(I64)],
    "sfb_frame": [P, P, P, I64, D, P, ctypes.POINTER(Camera_t), ctypes.POINTER(RenderOptions_t),
                  I32, P, P, P, P, P],
    "sfb_knn": [P, P, I64, I32, P, P],
    "sfb_nn_distance": [P, P, I64, I32, P],
    "sfb_local_pca": [P, P, I64, I32, P, D, D, P, P, P, P],
    "sfb_ply_decode": [P, P, I64, I32, P, P, P, P],
    "sfb_spl1_decode": [P, P, I64, P, P, P, P, P, P],
    "sfb_spl1_encode": [P, ctypes.POINTER(Splats_t), P],
    "sfb_render_backward": [P, ctypes.POINTER(Splats_t), ctypes.POINTER(Camera_t),
                            ctypes.POINTER(RenderOptions_t), I32, P, P, P, P, P, P, P, P],
    "sfb_render_rgba": [P, ctypes.POINTER(Splats_t), ctypes.POINTER(Camera_t),
                        ctypes.POINTER(RenderOptions_t), ctypes.POINTER(Shading_t), P, P],
    "sfb_frame_rgba": [P, P, P, I64, D, P, ctypes.POINTER(Camera_t),
                       ctypes.POINTER(RenderOptions_t), ctypes.POINTER(Shading_t), P, P],
}

_lib = None
_lock = threading.Lock()
_contexts = {}


def load_library():
    """dlopen libsfb200.so (no GPU needed to load) and declare every symbol."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_char_p if name == "sfb_last_error" else ctypes.c_int
        _lib = lib
    return _lib


class SfbError(RuntimeError):
    pass


class Context:
    """One library context per CUDA device (stream set per call)."""

    def __init__(self, device: int):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2409_16504_b200 needs a CUDA device (B200); "
                               "there is no CPU fallback")
        self.lib = load_library()
        self.device = device
        h = P()
        rc = self.lib.sfb_ctx_create(device, ctypes.byref(h))
        if rc != SFB_OK:
            raise SfbError(f"sfb_ctx_create failed ({rc})")
        self.handle = h
        self.lock = threading.RLock()
        self.net_token = None

    def call(self, name: str, *args):
        """Run one entry point on torch's current stream. The context's scratch
        arena is reused by every call, so the library orders a call issued on
        a different stream after the previous call's work (an event recorded
        at the end of each call, waited on when the stream changes); the lock
        keeps set-stream + call atomic across host threads."""
        import torch
        stream = torch.cuda.current_stream(self.device).cuda_stream
        with self.lock:
            self.lib.sfb_set_stream(self.handle, P(stream))
            rc = getattr(self.lib, name)(self.handle, *args)
            msg = self.lib.sfb_last_error(self.handle).decode(errors="replace") if rc else ""
        if rc != SFB_OK:
            if rc == SFB_ERR_ARG:
                raise ValueError(msg)
            raise SfbError(f"{name}: {msg} (code {rc})")

    def set_timing(self, on: bool) -> None:
        self.lib.sfb_set_timing(self.handle, int(bool(on)))

    def stage_times(self) -> dict:
        """{stage name: ms} of the last call (needs set_timing(True))."""
        ids = (I32 * 16)()
        ms = (ctypes.c_float * 16)()
        n = I32(0)
        if self.lib.sfb_stage_times(self.handle, ids, ms, 16, ctypes.byref(n)) != SFB_OK:
            raise SfbError("sfb_stage_times failed")
        out = {}
        for i in range(n.value):
            name = STAGES.get(ids[i], str(ids[i]))
            out[name] = out.get(name, 0.0) + ms[i]
        return out

    def stats(self) -> dict:
        s = Stats_t()
        self.lib.sfb_get_stats(self.handle, ctypes.byref(s))
        return dict(kept=s.kept, runs=s.runs, fine_entries=s.fine_entries,
                    super_entries=s.super_entries, global_entries=s.global_entries,
                    voxels=list(s.voxels))


def context(device=None, lane: int = 0) -> Context:
    """Library context of (device, lane). Each lane owns its own scratch arena
    and frame graphs, so frames issued on different CUDA streams through
    different lanes run concurrently on one GPU."""
    import torch
    dev = torch.cuda.current_device() if device is None else int(device)
    with _lock:
        ctx = _contexts.get((dev, lane))
        if ctx is None:
            ctx = _contexts[(dev, lane)] = Context(dev)
    return ctx


def all_contexts() -> list:
    """Every library context created so far (all devices and lanes)."""
    with _lock:
        return list(_contexts.values())


def ptr(t) -> P:
    """Device pointer of a torch tensor (None -> NULL)."""
    return P(0) if t is None else P(t.data_ptr())
