"""paper_2507_19718_b200 -- B200-native GSCache hot path (arXiv 2507.19718): real-time fitting
and querying of the multi-level 3D-Gaussian path-space radiance cache.

Thin ctypes binding of ``libgscache.so`` (C ABI in ``include/gscache.h``).  Argument
marshalling only: every step of the path runs in the library's sm_100a kernels.  There is
no CPU fallback -- if the library is missing or no sm_100 device exists, calls raise.

Buffers may be torch tensors (CUDA or CPU), numpy arrays or raw integer pointers; CUDA
tensors are passed by device pointer, host buffers are staged by the library.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgscache.so")
MAX_LEVELS = 16
NGROUPS = 5
STATUS = {0: "GC_OK", 1: "GC_ERR_ARG", 2: "GC_ERR_STATE", 3: "GC_ERR_CUDA", 4: "GC_ERR_OOM",
          5: "GC_ERR_NCCL", 6: "GC_ERR_UNSUPPORTED"}

# Symbols include/gscache.h declares (checked by tests/test_abi.py).
EXPORTS = ["gc_default_hparams", "gc_create", "gc_destroy", "gc_reserve", "gc_fit", "gc_query",
           "gc_query_radiance", "gc_fit_query", "gc_set_deferred_step", "gc_flush",
           "gc_params", "gc_set_params", "gc_reset_schedule", "gc_grid", "gc_info",
           "gc_nccl_unique_id", "gc_set_comm", "gc_debug_enable_grads", "gc_debug_grads",
           "gc_debug_coef_grads", "gc_list_generation", "gc_set_level_weights", "gc_level_plan",
           "gc_comm_info", "gc_adam_state", "gc_set_adam_state", "gc_alg1_terminate", "gc_reinit",
           "gc_render", "gc_fit_image", "gc_query_dense", "gc_fit_dense", "gc_slab_plan",
           "gc_debug_cull", "gc_debug_levels", "gc_profile_enable", "gc_profile_read",
           "gc_last_error", "gc_status_string"]


class GCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class gc_hparams(C.Structure):
    _fields_ = [("lr", C.c_float * NGROUPS), ("weight_decay", C.c_float * NGROUPS),
                ("beta1", C.c_float), ("beta2", C.c_float), ("adam_eps", C.c_float),
                ("hdr_eps", C.c_float), ("loss_grad_mode", C.c_int), ("lr_schedule", C.c_int),
                ("cutoff_sigma", C.c_float), ("init_opacity", C.c_float),
                ("init_scale_factor", C.c_float), ("init_zcap", C.c_float),
                ("cells_per_axis", C.c_int * MAX_LEVELS), ("cell_edge_scale", C.c_float)]


class gc_fit_stats(C.Structure):
    _fields_ = [("n_in", C.c_int64), ("n_valid", C.c_int64), ("n_dropped", C.c_int64),
                ("step", C.c_int64), ("nonfinite_grads", C.c_int64), ("n_pairs", C.c_int64),
                ("n_candidates", C.c_int64), ("flags", C.c_int64), ("count", C.c_int64 * MAX_LEVELS),
                ("loss", C.c_double * MAX_LEVELS)]

    def as_dict(self, L=MAX_LEVELS):
        return dict(n_in=self.n_in, n_valid=self.n_valid, n_dropped=self.n_dropped,
                    step=self.step, nonfinite_grads=self.nonfinite_grads, n_pairs=self.n_pairs,
                    n_candidates=self.n_candidates, flags=self.flags, count=list(self.count)[:L],
                    loss=list(self.loss)[:L])


def pinned_stats() -> "gc_fit_stats":
    """A gc_fit_stats in page-locked host memory (the library then copies the statistics
    with one cudaMemcpyAsync instead of a host callback); falls back to pageable memory."""
    try:
        import torch
        buf = torch.empty(C.sizeof(gc_fit_stats), dtype=torch.uint8).pin_memory()
        st = gc_fit_stats.from_address(buf.data_ptr())
        st._buf = buf
        return st
    except Exception:
        return gc_fit_stats()


class gc_camera(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("view", C.c_float * 12), ("znear", C.c_float)]


def make_camera(width, height, fx, fy, cx, cy, view, znear=0.2) -> "gc_camera":
    """gc_camera from a 3x4 (or 12) world->camera matrix [R | t]."""
    c = gc_camera()
    c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.znear = int(width), int(height), fx, fy, cx, cy, znear
    for i, v in enumerate(np.asarray(view, np.float64).reshape(12)):
        c.view[i] = float(v)
    return c


class gc_opt_counters(C.Structure):
    _fields_ = [("t", C.c_int64), ("adam_step", C.c_int64 * MAX_LEVELS),
                ("beta1_pow", C.c_double * MAX_LEVELS), ("beta2_pow", C.c_double * MAX_LEVELS)]


class gc_level_params(C.Structure):
    _fields_ = [("count", C.c_int64), ("position", C.c_void_p), ("rotation", C.c_void_p),
                ("color", C.c_void_p), ("log_scale", C.c_void_p), ("opacity_logit", C.c_void_p)]


_lib = None


def lib():
    """Load libgscache.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        sig = {
            "gc_default_hparams": (None, [vp]),
            "gc_create": (i32, [i32, vp, vp, vp, vp, C.c_uint64, vp, i32, vp]),
            "gc_destroy": (i32, [vp]),
            "gc_reserve": (i32, [vp, i64, i64]),
            "gc_fit": (i32, [vp, vp, vp, vp, i64, vp, vp]),
            "gc_query": (i32, [vp, vp, vp, i32, i64, vp, vp]),
            "gc_query_radiance": (i32, [vp, vp, vp, i32, i64, vp, vp, vp, vp, vp]),
            "gc_fit_query": (i32, [vp, vp, vp, vp, i64, vp, vp, i32, i64, vp, vp, vp, vp, vp, vp]),
            "gc_set_deferred_step": (i32, [vp, i32]),
            "gc_flush": (i32, [vp, vp]),
            "gc_params": (i32, [vp, i32, vp, vp]),
            "gc_set_params": (i32, [vp, i32, vp, i32, vp]),
            "gc_reset_schedule": (i32, [vp]),
            "gc_grid": (i32, [vp, i32, vp, vp, vp]),
            "gc_info": (i32, [vp, vp, vp]),
            "gc_nccl_unique_id": (i32, [vp]),
            "gc_set_comm": (i32, [vp, vp, i32, i32, i32]),
            "gc_set_level_weights": (i32, [vp, vp]),
            "gc_level_plan": (i32, [i32, vp, i32, vp, vp, vp, vp]),
            "gc_comm_info": (i32, [vp, vp, vp, vp, vp, vp]),
            "gc_adam_state": (i32, [vp, i32, vp, vp, vp, vp]),
            "gc_reinit": (i32, [vp, vp, vp, vp, C.c_uint64]),
            "gc_render": (i32, [vp, vp, i32, vp, vp, vp]),
            "gc_query_dense": (i32, [vp, vp, vp, i32, i64, vp, vp]),
            "gc_fit_dense": (i32, [vp, vp, vp, i32, vp, i64, vp, vp]),
            "gc_slab_plan": (i32, [i32, vp, vp, vp, vp, vp, i32, vp]),
            "gc_fit_image": (i32, [vp, vp, vp, vp, vp, vp]),
            "gc_alg1_terminate": (i32, [vp, vp, i32, C.c_float, vp, vp, C.c_float, i64, vp, vp, vp, vp]),
            "gc_set_adam_state": (i32, [vp, i32, vp, vp, vp, vp]),
            "gc_debug_enable_grads": (i32, [vp, i32]),
            "gc_debug_grads": (i32, [vp, i32, vp, vp]),
            "gc_debug_coef_grads": (i32, [vp, i32, vp, vp]),
            "gc_list_generation": (i32, [vp, vp]),
            "gc_debug_cull": (i32, [vp, i32, vp, vp, i64, vp, vp]),
            "gc_debug_levels": (i32, [vp, vp, vp]),
            "gc_profile_enable": (i32, [vp, i32]),
            "gc_profile_read": (i32, [vp, vp, i64, vp, vp, i32, vp, i32]),
            "gc_last_error": (C.c_char_p, []),
            "gc_status_string": (C.c_char_p, [i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise GCError(st, lib().gc_last_error().decode())


def default_hparams(**over) -> gc_hparams:
    hp = gc_hparams()
    lib().gc_default_hparams(C.byref(hp))
    for k, v in over.items():
        if k in ("lr", "weight_decay"):
            for i, x in enumerate(v):
                getattr(hp, k)[i] = float(x)
        elif k == "cells_per_axis":
            for i, x in enumerate(v):
                hp.cells_per_axis[i] = int(x)
        else:
            setattr(hp, k, v)
    return hp


class _Buf:
    """Pointer + keep-alive for a torch tensor / numpy array of the required dtype."""

    def __init__(self, x, dtype, shape_last=None, writable=False):
        self.keep = None
        if x is None:
            self.ptr = None
            self.n = 0
            return
        try:
            import torch
            if isinstance(x, torch.Tensor):
                want = {np.float32: torch.float32, np.int32: torch.int32}[dtype]
                if x.dtype != want or not x.is_contiguous():
                    if writable:
                        raise TypeError(f"output tensor must be contiguous {want}")
                    x = x.to(want).contiguous()
                self.keep = x
                self.ptr = x.data_ptr()
                self.n = x.numel()
                return
        except ImportError:
            pass
        if isinstance(x, int):
            self.ptr, self.n = x, -1
            return
        a = np.asarray(x)
        if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
            if writable:
                raise TypeError("output array must be C-contiguous of the right dtype")
            a = np.ascontiguousarray(a, dtype=dtype)
        self.keep = a
        self.ptr = a.ctypes.data
        self.n = a.size


def _out_like(pos, S, out):
    """`out` or a new [S][3] float32 array on `pos`'s device."""
    if out is not None:
        return out
    try:
        import torch
        if isinstance(pos, torch.Tensor):
            return torch.empty((S, 3), dtype=torch.float32, device=pos.device)
    except ImportError:
        pass
    return np.empty((S, 3), np.float32)


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class GSCache:
    """Owning wrapper of a ``gc_cache`` handle; method names follow the C ABI."""

    def __init__(self, counts, init_pos, init_rgb, init_log_scale=None, seed=0, hparams=None,
                 device=0):
        counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
        self.L = len(counts)
        self.counts = counts.copy()
        self.hp = hparams if isinstance(hparams, gc_hparams) else default_hparams(**(hparams or {}))
        p = _Buf(init_pos, np.float32)
        r = _Buf(init_rgb, np.float32)
        s = _Buf(init_log_scale, np.float32)
        h = C.c_void_p()
        _check(lib().gc_create(self.L, counts.ctypes.data, p.ptr, r.ptr, s.ptr, C.c_uint64(seed),
                               C.addressof(self.hp), device, C.byref(h)))
        self.h = h
        self.device = device
        self.goff = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self._stats = pinned_stats()

    # ----------------------------------------------------- screen-space cache images (f1)
    def render(self, cam: "gc_camera", level=-1, with_T=False, stream=None):
        """gc_render: cache images [Lr][H][W][3] (torch CUDA tensor; Lr = L for level -1)."""
        import torch
        Lr = self.L if level < 0 else 1
        out = torch.empty((Lr, cam.height, cam.width, 3), dtype=torch.float32, device=f"cuda:{self.device}")
        T = torch.empty((Lr, cam.height, cam.width), dtype=torch.float32, device=out.device) if with_T else None
        _check(lib().gc_render(self.h, C.byref(cam), int(level), out.data_ptr(),
                               T.data_ptr() if T is not None else None, _stream_ptr(stream)))
        return (out, T) if with_T else out

    def fit_image(self, cam: "gc_camera", target, valid=None, stream=None, stats=None):
        """gc_fit_image: one optimisation step on per-level radiance images target
        [L][H][W][3] (CUDA f32) with optional valid [L][H][W] (CUDA u8)."""
        st = stats if stats is not None else self._stats
        _check(lib().gc_fit_image(self.h, C.byref(cam), target.data_ptr(),
                                  valid.data_ptr() if valid is not None else None,
                                  _stream_ptr(stream), C.addressof(st)))
        return st

    def reinit(self, init_pos, init_rgb, init_log_scale=None, seed=0):
        """gc_reinit: rebuild the cache in place from a new point cloud (morphology change)."""
        p = _Buf(init_pos, np.float32)
        r = _Buf(init_rgb, np.float32)
        s = _Buf(init_log_scale, np.float32)
        _check(lib().gc_reinit(self.h, p.ptr, r.ptr, s.ptr, C.c_uint64(seed)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                lib().gc_destroy(h)
            except Exception:
                pass
            self.h = None

    def destroy(self):
        self.__del__()

    # ---------------------------------------------------------------- hot path
    def reserve(self, S_fit=0, S_query=0):
        _check(lib().gc_reserve(self.h, int(S_fit), int(S_query)))

    def fit(self, pos, path_len, rgb, stream=None, stats: gc_fit_stats | None = None):
        """One gc_fit step.  Returns the gc_fit_stats struct (valid after stream sync)."""
        p, n, r = _Buf(pos, np.float32), _Buf(path_len, np.int32), _Buf(rgb, np.float32)
        S = n.n if n.n >= 0 else p.n // 3
        st = self._stats if stats is None else stats
        _check(lib().gc_fit(self.h, p.ptr, n.ptr, r.ptr, S, _stream_ptr(stream), C.addressof(st)))
        self._keep = (p, n, r)
        return st

    def fit_query(self, pos, path_len, rgb, qpos, qlen=None, qlevel=-1, attenuation=None,
                  beta=None, unbiased_rgb=None, out=None, stream=None,
                  stats: gc_fit_stats | None = None):
        """gc_fit_query: the frame's lookups (pre-step parameters) + one fit step.  Returns
        (out, stats)."""
        p, n, r = _Buf(pos, np.float32), _Buf(path_len, np.int32), _Buf(rgb, np.float32)
        S = n.n if n.n >= 0 else p.n // 3
        qp = _Buf(qpos, np.float32)
        Sq = qp.n // 3
        out = _out_like(qpos, Sq, out)
        o = _Buf(out, np.float32, writable=True)
        qn = _Buf(qlen, np.int32)
        at, be, un = (_Buf(attenuation, np.float32), _Buf(beta, np.float32),
                      _Buf(unbiased_rgb, np.float32))
        st = self._stats if stats is None else stats
        _check(lib().gc_fit_query(self.h, p.ptr, n.ptr, r.ptr, S, qp.ptr, qn.ptr, int(qlevel), Sq,
                                  at.ptr, be.ptr, un.ptr, o.ptr, _stream_ptr(stream), C.addressof(st)))
        self._keep = (p, n, r)
        self._keep_q = (qp, qn, o, at, be, un)
        return out, st

    def query(self, pos, path_len=None, level=-1, out=None, stream=None):
        """Cache lookup; returns `out` (allocated like `pos` if None)."""
        p = _Buf(pos, np.float32)
        S = p.n // 3
        out = _out_like(pos, S, out)
        o = _Buf(out, np.float32, writable=True)
        n = _Buf(path_len, np.int32)
        _check(lib().gc_query(self.h, p.ptr, n.ptr, int(level), S, o.ptr, _stream_ptr(stream)))
        self._keep_q = (p, n, o)
        return out

    def fit_dense(self, pos, path_len, rgb, level=-1, stream=None, stats=None):
        """gc_fit_dense (dense fit step on the tensor cores, row A8's backward) on CUDA tensors:
        pos [S][3] f32, path_len [S] i32 (or None with `level`), rgb [S][3] f32."""
        S = int(pos.shape[0])
        st = stats if stats is not None else self._stats
        _check(lib().gc_fit_dense(self.h, pos.data_ptr(), path_len.data_ptr() if path_len is not None else None,
                                  int(level), rgb.data_ptr(), S, _stream_ptr(stream), C.addressof(st)))
        return st

    def query_dense(self, pos, path_len=None, level=-1, out=None, stream=None):
        """gc_query_dense (tensor-core dense lookups, row A8) on CUDA tensors."""
        import torch
        S = int(pos.shape[0])
        if out is None:
            out = torch.empty((S, 3), dtype=torch.float32, device=pos.device)
        _check(lib().gc_query_dense(self.h, pos.data_ptr(), path_len.data_ptr() if path_len is not None else None,
                                    int(level), S, out.data_ptr(), _stream_ptr(stream)))
        return out

    def query_radiance(self, pos, path_len=None, level=-1, attenuation=None, beta=None,
                       unbiased_rgb=None, out=None, stream=None):
        """gc_query_radiance: lookup + natural-termination substitution + Eq. 3 scaling."""
        p = _Buf(pos, np.float32)
        S = p.n // 3
        out = _out_like(pos, S, out)
        o = _Buf(out, np.float32, writable=True)
        n = _Buf(path_len, np.int32)
        at, be, un = (_Buf(attenuation, np.float32), _Buf(beta, np.float32),
                      _Buf(unbiased_rgb, np.float32))
        _check(lib().gc_query_radiance(self.h, p.ptr, n.ptr, int(level), S, at.ptr, be.ptr, un.ptr,
                                       o.ptr, _stream_ptr(stream)))
        self._keep_q = (p, n, o, at, be, un)
        return out

    # ------------------------------------------------------------ params I/O
    def _level_struct(self, level, arrays):
        lp = gc_level_params()
        lp.count = int(self.counts[level])
        lp.position = arrays["position"].ctypes.data
        lp.rotation = arrays["rotation"].ctypes.data
        lp.color = arrays["color"].ctypes.data
        lp.log_scale = arrays["log_scale"].ctypes.data
        lp.opacity_logit = arrays["opacity_logit"].ctypes.data
        return lp

    def _empty_level(self, level):
        n = int(self.counts[level])
        return dict(position=np.empty((n, 3), np.float32), rotation=np.empty((n, 4), np.float32),
                    color=np.empty((n, 3), np.float32), log_scale=np.empty((n, 3), np.float32),
                    opacity_logit=np.empty((n, 1), np.float32))

    def params(self, level, stream=None):
        """Raw parameters of one level (numpy, paper layout P:444-448); synchronises."""
        a = self._empty_level(level)
        lp = self._level_struct(level, a)
        _check(lib().gc_params(self.h, level, C.byref(lp), _stream_ptr(stream)))
        self.synchronize(stream)
        return a

    def params_rows(self, level, stream=None):
        """[N][14] rows in paper order (oracle layout)."""
        a = self.params(level, stream)
        return np.concatenate([a["position"], a["rotation"], a["color"], a["log_scale"],
                               a["opacity_logit"]], axis=1)

    def set_params(self, level, arrays, reset_adam=False, stream=None):
        a = {k: np.ascontiguousarray(np.asarray(v, np.float32)) for k, v in arrays.items()}
        lp = self._level_struct(level, a)
        _check(lib().gc_set_params(self.h, level, C.byref(lp), int(bool(reset_adam)),
                                   _stream_ptr(stream)))
        self.synchronize(stream)

    def set_params_rows(self, level, rows, reset_adam=False):
        rows = np.asarray(rows, np.float32)
        self.set_params(level, dict(position=rows[:, 0:3], rotation=rows[:, 3:7],
                                    color=rows[:, 7:10], log_scale=rows[:, 10:13],
                                    opacity_logit=rows[:, 13:14]), reset_adam)

    @staticmethod
    def _rows(a):
        return np.concatenate([a["position"], a["rotation"], a["color"], a["log_scale"],
                               a["opacity_logit"]], axis=1)

    @staticmethod
    def _split(rows):
        rows = np.ascontiguousarray(np.asarray(rows, np.float32))
        return {k: np.ascontiguousarray(rows[:, a:b]) for k, (a, b) in
                dict(position=(0, 3), rotation=(3, 7), color=(7, 10), log_scale=(10, 13),
                     opacity_logit=(13, 14)).items()}

    def adam_state(self, level, stream=None):
        """(m rows [N][14], v rows [N][14], counters) of one level (gc_adam_state)."""
        m, v = self._empty_level(level), self._empty_level(level)
        lm, lv = self._level_struct(level, m), self._level_struct(level, v)
        ctr = gc_opt_counters()
        _check(lib().gc_adam_state(self.h, level, C.byref(lm), C.byref(lv), C.byref(ctr), _stream_ptr(stream)))
        self.synchronize(stream)
        return self._rows(m), self._rows(v), dict(t=ctr.t, adam_step=list(ctr.adam_step),
                                                  beta1_pow=list(ctr.beta1_pow), beta2_pow=list(ctr.beta2_pow))

    def set_adam_state(self, level, m_rows, v_rows, counters=None, stream=None):
        m, v = self._split(m_rows), self._split(v_rows)
        lm, lv = self._level_struct(level, m), self._level_struct(level, v)
        ctr = None
        if counters is not None:
            ctr = gc_opt_counters()
            ctr.t = int(counters["t"])
            for l in range(MAX_LEVELS):
                ctr.adam_step[l] = int(counters["adam_step"][l])
                ctr.beta1_pow[l] = float(counters["beta1_pow"][l])
                ctr.beta2_pow[l] = float(counters["beta2_pow"][l])
        _check(lib().gc_set_adam_state(self.h, level, C.byref(lm), C.byref(lv),
                                       C.byref(ctr) if ctr is not None else None, _stream_ptr(stream)))
        self.synchronize(stream)

    def set_deferred_step(self, on=True):
        """gc_set_deferred_step: leave each fit's optimizer half pending for the next call."""
        _check(lib().gc_set_deferred_step(self.h, 1 if on else 0))

    def flush(self, stream=None):
        """gc_flush: complete a pending (deferred) optimizer step on `stream`."""
        _check(lib().gc_flush(self.h, _stream_ptr(stream)))

    def reset_schedule(self):
        _check(lib().gc_reset_schedule(self.h))

    def grid(self, level):
        o = (C.c_double * 3)()
        ic = (C.c_double * 3)()
        d = (C.c_int32 * 3)()
        _check(lib().gc_grid(self.h, level, o, ic, d))
        return np.array(o[:]), np.array(ic[:]), np.array(d[:], np.int32)

    def grids(self):
        return [self.grid(l) for l in range(self.L)]

    def set_comm(self, uid: bytes, rank: int, world: int, mode: int = 0):
        buf = C.create_string_buffer(uid, 128) if uid is not None else None
        _check(lib().gc_set_comm(self.h, buf, rank, world, mode))

    def set_level_weights(self, weights=None):
        """Level weights of the level-sharded plan (mode 1); None = per-level Gaussian share."""
        w = None if weights is None else (C.c_double * self.L)(*[float(v) for v in weights])
        _check(lib().gc_set_level_weights(self.h, w))

    def comm_info(self):
        v = [C.c_int() for _ in range(5)]
        _check(lib().gc_comm_info(self.h, *[C.byref(x) for x in v]))
        return dict(mode=v[0].value, rank=v[1].value, world=v[2].value,
                    owned_levels=[l for l in range(self.L) if (v[3].value >> l) & 1],
                    group_size=v[4].value)

    # ----------------------------------------------------------------- debug
    def debug_enable_grads(self, on=True, coef=False):
        """Bit 0 (on): raw 14-parameter gradients; bit 1 (coef): the coefficient-gradient
        snapshot of the unchanged (lite) hot path."""
        _check(lib().gc_debug_enable_grads(self.h, int(bool(on)) | (2 if coef else 0)))

    def debug_coef_grads(self, level, stream=None):
        """[n][12] coefficient gradients of the last fit (dmu, dA00 dA11 dA22 dA01 dA02 dA12,
        dv), not divided by 3 k_l."""
        out = np.empty((int(self.counts[level]), 12), np.float32)
        _check(lib().gc_debug_coef_grads(self.h, level, out.ctypes.data, _stream_ptr(stream)))
        return out

    def list_generation(self):
        g = C.c_uint64()
        _check(lib().gc_list_generation(self.h, C.byref(g)))
        return g.value

    def debug_grads_rows(self, level, stream=None):
        a = self._empty_level(level)
        lp = self._level_struct(level, a)
        _check(lib().gc_debug_grads(self.h, level, C.byref(lp), _stream_ptr(stream)))
        self.synchronize(stream)
        return np.concatenate([a["position"], a["rotation"], a["color"], a["log_scale"],
                               a["opacity_logit"]], axis=1)

    def debug_cull(self, level, stream=None):
        o, ic, d = self.grid(level)
        cells = int(d[0]) * int(d[1]) * int(d[2])
        off = np.empty(cells + 1, np.int32)
        n = C.c_int64()
        lib().gc_debug_cull(self.h, level, off.ctypes.data, None, 0, C.byref(n), _stream_ptr(stream))
        idx = np.empty(max(n.value, 1), np.int32)
        _check(lib().gc_debug_cull(self.h, level, off.ctypes.data, idx.ctypes.data, idx.size,
                                   C.byref(n), _stream_ptr(stream)))
        return off, idx[:n.value]

    def debug_levels(self, S, stream=None):
        out = np.empty(S, np.int32)
        _check(lib().gc_debug_levels(self.h, out.ctypes.data, _stream_ptr(stream)))
        return out

    def profile_enable(self, on=True):
        _check(lib().gc_profile_enable(self.h, int(bool(on))))

    def profile_read(self, reset=True):
        names = C.create_string_buffer(4096)
        ms = (C.c_double * 64)()
        ln = (C.c_int64 * 64)()
        nk = C.c_int()
        _check(lib().gc_profile_read(self.h, names, 4096, ms, ln, 64, C.byref(nk), int(reset)))
        keys = names.value.decode().split(";") if nk.value else []
        return {k: (ms[i], ln[i]) for i, k in enumerate(keys)}

    def synchronize(self, stream=None):
        try:
            import torch
            if stream is not None:
                stream.synchronize()
            else:
                torch.cuda.synchronize(self.device)
        except Exception:
            pass


def alg1_terminate(sigma, n, C_, q, beta=None, eps=1e-6, stream=None):
    """gc_alg1_terminate on torch CUDA tensors: sigma [P][nmax][3] f32, n [P] i32, q [P] f32,
    beta [P] f32 or None -> (terminate i32 [P], tr_out f32 [P][3], beta_next f32 [P])."""
    import torch
    P, nmax = int(sigma.shape[0]), int(sigma.shape[1])
    dev = sigma.device
    term = torch.empty(P, dtype=torch.int32, device=dev)
    tr = torch.empty((P, 3), dtype=torch.float32, device=dev)
    bn = torch.empty(P, dtype=torch.float32, device=dev)
    _check(lib().gc_alg1_terminate(sigma.data_ptr(), n.data_ptr(), nmax, float(C_),
                                   beta.data_ptr() if beta is not None else None, q.data_ptr(),
                                   float(eps), P, term.data_ptr(), tr.data_ptr(), bn.data_ptr(),
                                   _stream_ptr(stream)))
    return term, tr, bn


def slab_plan(counts, means_x, grids, world: int):
    """gc_slab_plan (host): [levels][512] column -> rank table of the owner-computes mode."""
    counts = np.ascontiguousarray(counts, np.int64)
    L = len(counts)
    mx = np.ascontiguousarray(means_x, np.float32)
    o = np.ascontiguousarray([g[0] for g in grids], np.float64)
    ic = np.ascontiguousarray([g[1] for g in grids], np.float64)
    dm = np.ascontiguousarray([g[2] for g in grids], np.int32)
    out = np.empty((L, 512), np.int32)
    st = lib().gc_slab_plan(L, counts.ctypes.data, mx.ctypes.data, o.ctypes.data, ic.ctypes.data,
                            dm.ctypes.data, int(world), out.ctypes.data)
    if st != 0:
        raise GCError(st, "gc_slab_plan: bad arguments")
    return out


def level_plan(weights, world: int):
    """gc_level_plan (pure host function): returns (group_of_level, [(first_rank, size)])."""
    L = len(weights)
    w = (C.c_double * L)(*[float(v) for v in weights])
    gl = (C.c_int32 * L)()
    fr = (C.c_int32 * L)()
    gs = (C.c_int32 * L)()
    ng = C.c_int()
    st = lib().gc_level_plan(L, w, world, gl, fr, gs, C.byref(ng))
    if st != 0:
        raise GCError(st, "gc_level_plan: bad arguments")
    return list(gl), [(fr[g], gs[g]) for g in range(ng.value)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().gc_nccl_unique_id(buf))
    return buf.raw


# module-level names matching the C ABI
def gc_create(counts, init_pos, init_rgb, init_log_scale=None, seed=0, hparams=None, device=0):
    return GSCache(counts, init_pos, init_rgb, init_log_scale, seed, hparams, device)


def gc_fit(cache: GSCache, pos, path_len, rgb, stream=None):
    return cache.fit(pos, path_len, rgb, stream)


def gc_fit_query(cache: GSCache, pos, path_len, rgb, qpos, qlen=None, qlevel=-1, out=None,
                 stream=None):
    return cache.fit_query(pos, path_len, rgb, qpos, qlen, qlevel, out=out, stream=stream)


def gc_query(cache: GSCache, pos, path_len=None, level=-1, out=None, stream=None):
    return cache.query(pos, path_len, level, out, stream)


def gc_params(cache: GSCache, level):
    return cache.params(level)
