"""Thin ctypes binding of libwino.so (include/wino.h).

Argument marshalling only: every stage of the layer runs in the CUDA kernels
behind the C ABI.  The module-level functions carry the C names
(``wino_plan_create``, ``wino_filter_transform``, ``wino_forward``, ...);
``Plan`` is a convenience wrapper over them.  Tensors are torch CUDA tensors
(fp32, contiguous) and are passed as raw device pointers; PyTorch provides
device memory and streams only.

There is no fallback: if libwino.so is missing or fails to load this module
raises, and a call on a machine without a usable device returns
WINO_ERR_CUDA through the ABI.
"""
from __future__ import annotations

import ctypes
import os
import json
from pathlib import Path
from typing import Optional, Sequence

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libwino.so"

WINO_OK, WINO_ERR_ARG, WINO_ERR_SHAPE, WINO_ERR_POINTS, WINO_ERR_SYNTH = 0, 1, 2, 3, 4
WINO_ERR_STATE, WINO_ERR_UNSUPPORTED, WINO_ERR_CUDA, WINO_ERR_NOMEM = 5, 6, 7, 8
STATUS_NAMES = {0: "WINO_OK", 1: "WINO_ERR_ARG", 2: "WINO_ERR_SHAPE", 3: "WINO_ERR_POINTS",
                4: "WINO_ERR_SYNTH", 5: "WINO_ERR_STATE", 6: "WINO_ERR_UNSUPPORTED",
                7: "WINO_ERR_CUDA", 8: "WINO_ERR_NOMEM"}
WINO_GEMM_AUTO, WINO_GEMM_FFMA, WINO_GEMM_1XTF32, WINO_GEMM_3XTF32, WINO_GEMM_3XF16 = 0, 1, 2, 3, 4
WINO_FUSE_NONE, WINO_FUSE_L2_CHUNK = 0, 4
WINO_ACT_NONE, WINO_ACT_RELU = 0, 1

EXPORTS = ["wino_plan_create", "wino_plan_create_ex", "wino_plan_create_nd", "wino_plan_destroy", "wino_filter_transform",
           "wino_forward", "wino_forward_ex", "wino_forward_host", "wino_plan_out_dims", "wino_plan_sizes",
           "wino_plan_info", "wino_filter_buffer", "wino_filter_mark_ready", "wino_workspace",
           "wino_profile_enable", "wino_profile_read", "wino_synthesize", "wino_get_transforms",
           "wino_last_error", "wino_version"]


class WinoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libwino.so (build it first with paper_1611_06565_b200._build)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError("libwino.so not built: run `python -m paper_1611_06565_b200._build` "
                              "(or __graft_entry__.build())")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64p, i32p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
        sz, szp, dp = ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double)
        c_int = ctypes.c_int
        sig = {
            "wino_plan_create": [ctypes.POINTER(vp), c_int, i64p, c_int, c_int, c_int, c_int, c_int, i32p],
            "wino_plan_create_ex": [ctypes.POINTER(vp), c_int, i64p, c_int, c_int, c_int, c_int, c_int,
                                    i32p, ctypes.c_char_p, c_int, c_int, c_int],
            "wino_plan_create_nd": [ctypes.POINTER(vp), c_int, i64p, i32p, i32p, c_int, c_int, c_int, i32p,
                                    c_int, c_int],
            "wino_plan_destroy": [vp],
            "wino_filter_transform": [vp, vp, vp],
            "wino_forward": [vp, vp, vp, c_int, vp],
            "wino_forward_ex": [vp, vp, vp, c_int, vp, c_int, vp],
            "wino_forward_host": [vp, vp, vp, c_int, vp],
            "wino_plan_out_dims": [vp, i64p],
            "wino_plan_sizes": [vp, szp, szp],
            "wino_plan_info": [vp, i64p],
            "wino_filter_buffer": [vp, ctypes.POINTER(vp), szp],
            "wino_filter_mark_ready": [vp],
            "wino_workspace": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)],
            "wino_profile_enable": [vp, c_int],
            "wino_profile_read": [vp, dp, i32p],
            "wino_synthesize": [c_int, c_int, ctypes.c_char_p, dp, dp, dp, ctypes.c_char_p, sz],
            "wino_get_transforms": [vp, dp, dp, dp, ctypes.c_char_p, sz],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = c_int
        L.wino_last_error.restype = ctypes.c_char_p
        L.wino_last_error.argtypes = []
        L.wino_version.restype = ctypes.c_char_p
        L.wino_version.argtypes = []
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != WINO_OK:
        raise WinoError(st, lib().wino_last_error().decode())


def _i64arr(v):
    return (ctypes.c_int64 * len(v))(*[int(a) for a in v])


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev_ptr(t, name):
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("%s must be a contiguous CUDA tensor" % name)
    import torch
    if t.dtype != torch.float32:
        raise ValueError("%s must be float32" % name)
    return t.data_ptr()


# ------------------------------------------------------------- C-named calls
def wino_version() -> str:
    return lib().wino_version().decode()


def wino_last_error() -> str:
    return lib().wino_last_error().decode()


def wino_synthesize(m: int, r: int, points: Optional[str] = None) -> dict:
    """Host-only exact synthesis: dict with exact rational strings and doubles."""
    a = m + r - 1
    AT = (ctypes.c_double * (m * a))()
    G = (ctypes.c_double * (a * r))()
    BT = (ctypes.c_double * (a * a))()
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().wino_synthesize(m, r, points.encode() if points else None, AT, G, BT, buf, len(buf)))
    d = json.loads(buf.value.decode())
    d["AT_f64"] = [list(AT[i * a:(i + 1) * a]) for i in range(m)]
    d["G_f64"] = [list(G[i * r:(i + 1) * r]) for i in range(a)]
    d["BT_f64"] = [list(BT[i * a:(i + 1) * a]) for i in range(a)]
    return d


def wino_plan_create_ex(N, dims, m, r, C, K, batch, padding=None, points=None, gemm_mode=0, fuse=0,
                        device=-1) -> int:
    h = ctypes.c_void_p()
    pad = (ctypes.c_int * N)(*([0] * N if padding is None else [int(p) for p in padding]))
    _check(lib().wino_plan_create_ex(ctypes.byref(h), int(N), _i64arr(dims), int(m), int(r), int(C),
                                     int(K), int(batch), pad, points.encode() if points else None,
                                     int(gemm_mode), int(fuse), int(device)))
    return h.value


def wino_plan_create_nd(N, dims, m, r, C, K, batch, padding=None, gemm_mode=0, device=-1) -> int:
    """Per-axis (m_n, r_n) plan (include/wino.h wino_plan_create_nd)."""
    h = ctypes.c_void_p()
    pad = (ctypes.c_int * N)(*([0] * N if padding is None else [int(p) for p in padding]))
    mv = (ctypes.c_int * N)(*[int(v) for v in m])
    rv = (ctypes.c_int * N)(*[int(v) for v in r])
    _check(lib().wino_plan_create_nd(ctypes.byref(h), int(N), _i64arr(dims), mv, rv, int(C), int(K), int(batch),
                                     pad, int(gemm_mode), int(device)))
    return h.value


def wino_plan_create(N, dims, m, r, C, K, batch, padding=None) -> int:
    h = ctypes.c_void_p()
    pad = (ctypes.c_int * N)(*([0] * N if padding is None else [int(p) for p in padding]))
    _check(lib().wino_plan_create(ctypes.byref(h), int(N), _i64arr(dims), int(m), int(r), int(C), int(K),
                                  int(batch), pad))
    return h.value


def wino_plan_destroy(plan: int) -> None:
    _check(lib().wino_plan_destroy(plan))


def wino_filter_transform(plan: int, g, stream=None) -> None:
    _check(lib().wino_filter_transform(plan, _dev_ptr(g, "g"), _stream_ptr(stream)))


def wino_forward(plan: int, x, y, B: int, stream=None) -> None:
    _check(lib().wino_forward(plan, _dev_ptr(x, "x"), _dev_ptr(y, "y"), int(B), _stream_ptr(stream)))


def wino_forward_ex(plan: int, x, y, B: int, bias=None, activation: int = WINO_ACT_NONE, stream=None) -> None:
    """Eq. (2) with bias b[k] (CUDA float32 [K] or None) and activation f."""
    bp = None if bias is None else _dev_ptr(bias, "bias")
    _check(lib().wino_forward_ex(plan, _dev_ptr(x, "x"), _dev_ptr(y, "y"), int(B), bp, int(activation),
                                 _stream_ptr(stream)))


def wino_forward_host(plan: int, x_host, y_host, B: int, stream=None) -> None:
    """x_host / y_host: CPU float32 contiguous tensors (pin_memory() for speed)."""
    import torch
    for t, n in ((x_host, "x_host"), (y_host, "y_host")):
        if t.is_cuda or not t.is_contiguous() or t.dtype != torch.float32:
            raise ValueError("%s must be a contiguous CPU float32 tensor" % n)
    _check(lib().wino_forward_host(plan, x_host.data_ptr(), y_host.data_ptr(), int(B), _stream_ptr(stream)))


def wino_plan_out_dims(plan: int, N: int):
    out = (ctypes.c_int64 * N)()
    _check(lib().wino_plan_out_dims(plan, out))
    return tuple(out)


def wino_plan_sizes(plan: int):
    ws, fb = ctypes.c_size_t(), ctypes.c_size_t()
    _check(lib().wino_plan_sizes(plan, ctypes.byref(ws), ctypes.byref(fb)))
    return ws.value, fb.value


INFO_KEYS = ["N", "m", "r", "alpha", "C", "K", "batch", "T_per_sample", "T_stride", "n_points", "K_stride",
             "gemm_mode", "fuse", "n_blk", "k_chunk", "chunk_slabs", "gemm_variant", "in_slab_tiles",
             "in_planes_per_cta", "axis_mode", "tiny", "launches", "in_bands", "fold", "fold_mode"]


def wino_plan_info(plan: int) -> dict:
    info = (ctypes.c_int64 * len(INFO_KEYS))()
    _check(lib().wino_plan_info(plan, info))
    return dict(zip(INFO_KEYS, list(info)))


def wino_filter_buffer(plan: int):
    p, n = ctypes.c_void_p(), ctypes.c_size_t()
    _check(lib().wino_filter_buffer(plan, ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def wino_filter_mark_ready(plan: int) -> None:
    _check(lib().wino_filter_mark_ready(plan))


def wino_workspace(plan: int):
    v, m = ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().wino_workspace(plan, ctypes.byref(v), ctypes.byref(m)))
    return v.value, m.value


def wino_profile_enable(plan: int, enable: bool = True) -> None:
    _check(lib().wino_profile_enable(plan, int(bool(enable))))


def wino_profile_read(plan: int):
    ms = (ctypes.c_double * 3)()
    calls = ctypes.c_int()
    _check(lib().wino_profile_read(plan, ms, ctypes.byref(calls)))
    return list(ms), calls.value


def wino_get_transforms(plan: int) -> dict:
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib().wino_get_transforms(plan, None, None, None, buf, len(buf)))
    return json.loads(buf.value.decode())


# ------------------------------------------------------------- torch views
class _CAI:
    def __init__(self, ptr, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr: int, shape, device=None):
    """A torch CUDA float32 tensor aliasing plan-owned device memory."""
    import torch
    return torch.as_tensor(_CAI(ptr, shape), device=device or "cuda")


def _nvtx_on() -> bool:
    return os.environ.get("WINO_NVTX", "0") not in ("", "0")


# ------------------------------------------------------------- Plan
class Plan:
    """One N-D Winograd conv layer F(m^N, r^N) on one GPU.

    Plan(N, dims, m, r, C, K, batch, padding=None, points=None, gemm_mode=0, fuse=0, device=-1)

    m and r may be per-axis sequences (F(m_1 x .. x m_N, r_1 x .. x r_N),
    wino_plan_create_nd); then g is [K][C][r_1]..[r_N] and points / fuse
    must be left at their defaults.
    """

    def __init__(self, N: int, dims: Sequence[int], m: int, r: int, C: int, K: int, batch: int,
                 padding: Optional[Sequence[int]] = None, points: Optional[str] = None,
                 gemm_mode: int = WINO_GEMM_AUTO, fuse: int = 0, device: int = -1):
        self.N, self.dims, self.m, self.r, self.C, self.K, self.batch = N, tuple(dims), m, r, C, K, batch
        self.padding = tuple(padding) if padding is not None else (0,) * N
        if isinstance(m, (list, tuple)) or isinstance(r, (list, tuple)):
            mv = tuple(m) if isinstance(m, (list, tuple)) else (m,) * N
            rv = tuple(r) if isinstance(r, (list, tuple)) else (r,) * N
            if len(mv) != N or len(rv) != N:
                raise ValueError("per-axis m and r need N entries")
            if points is not None or fuse:
                raise ValueError("per-axis plans take the default points and no fusion")
            self.m, self.r = mv, rv
            self.h = wino_plan_create_nd(N, dims, mv, rv, C, K, batch, self.padding, gemm_mode, device)
        else:
            self.h = wino_plan_create_ex(N, dims, m, r, C, K, batch, self.padding, points, gemm_mode, fuse, device)
        self.out_dims = wino_plan_out_dims(self.h, N)
        self.info = wino_plan_info(self.h)

    @property
    def launches_per_forward(self) -> int:
        """Kernel launches of one full-batch forward (wino_plan_info)."""
        return int(self.info["launches"])

    # The C ABI takes raw pointers and trusts the sizes: every tensor is
    # checked against the plan's shapes here, before its pointer is passed.
    def _kernel_dims(self):
        return tuple(self.r) if isinstance(self.r, tuple) else (self.r,) * self.N

    def _check_x(self, x, name="x"):
        if x.dim() != self.N + 2 or tuple(x.shape[1:]) != (self.C,) + self.dims:
            raise ValueError("%s has shape %s, the plan needs (B, %d, %s)" %
                             (name, tuple(x.shape), self.C, ", ".join(map(str, self.dims))))
        if not 1 <= x.shape[0] <= self.batch:
            raise ValueError("%s batch %d outside 1..%d (planned batch)" % (name, x.shape[0], self.batch))

    def _check_y(self, y, B, name="y"):
        want = (B, self.K) + tuple(self.out_dims)
        if tuple(y.shape) != want:
            raise ValueError("%s has shape %s, the plan writes %s" % (name, tuple(y.shape), want))

    def filter_transform(self, g, stream=None) -> None:
        want = (self.K, self.C) + self._kernel_dims()
        if tuple(g.shape) != want:
            raise ValueError("g has shape %s, the plan needs %s" % (tuple(g.shape), want))
        wino_filter_transform(self.h, g, stream)

    def forward(self, x, y=None, stream=None, bias=None, relu=False):
        """y = conv(x) (+ bias[k]) (then ReLU): Eq. (2) with b and f optional."""
        import torch
        self._check_x(x)
        B = x.shape[0]
        if y is None:
            y = torch.empty((B, self.K) + tuple(self.out_dims), device=x.device, dtype=torch.float32)
        self._check_y(y, B)
        if bias is not None and tuple(bias.shape) != (self.K,):
            raise ValueError("bias has shape %s, the plan needs (%d,)" % (tuple(bias.shape), self.K))
        nvtx = _nvtx_on()
        if nvtx:   # WINO_NVTX=1: an NVTX range around the ABI call (nsys / ncu --nvtx timelines)
            torch.cuda.nvtx.range_push("wino_forward N=%d F(%s,%s) C=%d K=%d B=%d" % (self.N, self.m, self.r, self.C, self.K, B))
        try:
            if bias is None and not relu:
                wino_forward(self.h, x, y, B, stream)
            else:
                wino_forward_ex(self.h, x, y, B, bias, WINO_ACT_RELU if relu else WINO_ACT_NONE, stream)
        finally:
            if nvtx:
                torch.cuda.nvtx.range_pop()
        return y

    def forward_host(self, x_host, y_host, stream=None) -> None:
        self._check_x(x_host, "x_host")
        self._check_y(y_host, x_host.shape[0], "y_host")
        wino_forward_host(self.h, x_host, y_host, x_host.shape[0], stream)

    def filter_tensor(self):
        """The U buffer (U_hi | U_lo) as a flat float32 CUDA tensor (for NCCL broadcast)."""
        ptr, nbytes = wino_filter_buffer(self.h)
        return device_view(ptr, (nbytes // 4,))

    def mark_ready(self) -> None:
        wino_filter_mark_ready(self.h)

    def workspace(self):
        """(V [P][C][T_s], M [P][K][T_s]) views of the unfused workspace."""
        v, m = wino_workspace(self.h)
        P, Ts = self.info["n_points"], self.info["T_stride"]
        return device_view(v, (P, self.C, Ts)), device_view(m, (P, self.K, Ts))

    def transforms(self) -> dict:
        return wino_get_transforms(self.h)

    def profile(self, enable=True):
        wino_profile_enable(self.h, enable)

    def profile_read(self):
        return wino_profile_read(self.h)

    def sizes(self):
        return wino_plan_sizes(self.h)

    def close(self) -> None:
        if getattr(self, "h", None):
            wino_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
