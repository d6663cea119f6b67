"""ctypes binding of libfsr.so (include/fsr.h).

This is the one place the Python package touches native code.  There is no
fallback: if the shared library is missing or no CUDA device is present,
every call raises.
"""

from __future__ import annotations

import ctypes
import mmap
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSR_LIBFSR overrides the library path (used to A/B kernel build variants)
LIB_PATH = os.environ.get("FSR_LIBFSR") or os.path.join(_HERE, "libfsr.so")

FSR_OK, FSR_EINVAL, FSR_ENOSAMPLES, FSR_ECUDA, FSR_EUNSUPPORTED = 0, 1, 2, 3, 4
REDUCER = {"tree": 0, "linear": 1}
PRECISION = {"fp64": 0, "fp32": 1, "fp32_unguarded": 2}
ARGMAX = {"shfl": 0, "smem": 1, "redux": 2}
KERNEL = {"auto": 0, "warp": 1, "pair": 2}


class FsrParamsC(ctypes.Structure):
    _fields_ = [
        ("block", ctypes.c_int32),
        ("border", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("reducer", ctypes.c_int32),
        ("early_stop", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("argmax_impl", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("rho", ctypes.c_double),
        ("gamma", ctypes.c_double),
        ("guard_tau", ctypes.c_double),
        ("guard_kappa", ctypes.c_double),
    ]


class FsrStatsC(ctypes.Structure):
    _fields_ = [
        ("blocks", ctypes.c_int64),
        ("rerun_blocks", ctypes.c_int64),
        ("empty_blocks", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("kernel_ms", ctypes.c_double),
        ("main_ms", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()


def load():
    """Load libfsr.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (make -C paper_2202_13926_b200/csrc); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        pp = ctypes.POINTER(FsrParamsC)
        L.fsr_params_init.argtypes = [pp]
        L.fsr_params_init.restype = None
        L.fsr_params_validate.argtypes = [pp, ctypes.c_char_p, ctypes.c_int]
        L.fsr_params_validate.restype = ctypes.c_int
        L.fsr_engine_create.argtypes = [P, i32, ctypes.POINTER(P)]
        L.fsr_engine_create.restype = ctypes.c_int
        L.fsr_engine_destroy.argtypes = [P]
        L.fsr_engine_destroy.restype = None
        L.fsr_last_error.argtypes = [P]
        L.fsr_last_error.restype = ctypes.c_char_p
        L.fsr_status_string.argtypes = [ctypes.c_int]
        L.fsr_status_string.restype = ctypes.c_char_p
        L.fsr_pin_host.argtypes = [P, ctypes.c_size_t]
        L.fsr_pin_host.restype = ctypes.c_int
        L.fsr_unpin_host.argtypes = [P]
        L.fsr_unpin_host.restype = ctypes.c_int
        L.fsr_abi_version.restype = i32
        L.fsr_reconstruct_f64.argtypes = [P, pp, P, P, i64, i64, P, P, P]
        L.fsr_reconstruct_f64.restype = ctypes.c_int
        L.fsr_reconstruct_f32.argtypes = [P, pp, P, P, i64, i64, P, P, P]
        L.fsr_reconstruct_f32.restype = ctypes.c_int
        dbl = ctypes.c_double
        for io in ("f32", "f64"):
            f = getattr(L, f"fsr_reconstruct_rows_{io}")
            f.argtypes = [P, pp, P, P, i64, i64, i64, i64, dbl, P]
            f.restype = ctypes.c_int
            f = getattr(L, f"fsr_reconstruct_device_{io}")
            f.argtypes = [P, pp, P, i64, P, i64, i64, i64, i64, i64, P, i64, dbl, P]
            f.restype = ctypes.c_int
        L.fsr_iterate_spectra.argtypes = [P, pp, i64, i32, P, P, P, P, P, P, P, P, P]
        L.fsr_iterate_spectra.restype = ctypes.c_int
        L.fsr_spatial_oracle.argtypes = [P, i32, i32, ctypes.c_double, i64, P, P, P, P, P, P, P, P, P]
        L.fsr_spatial_oracle.restype = ctypes.c_int
        L.fsr_quarter_sample_device.argtypes = [P, P, i64, i64, i64, ctypes.c_uint64, P, i64, P, i64, P]
        L.fsr_quarter_sample_device.restype = ctypes.c_int
        L.fsr_sq_error_device.argtypes = [P, P, i64, P, i64, i64, i64, P, P]
        L.fsr_sq_error_device.restype = ctypes.c_int
        L.fsr_last_stats.argtypes = [P, ctypes.POINTER(FsrStatsC)]
        L.fsr_last_stats.restype = ctypes.c_int
        _lib = L
        return L


EXPORTED = ["fsr_params_init", "fsr_params_validate", "fsr_engine_create", "fsr_engine_destroy",
            "fsr_last_error", "fsr_status_string", "fsr_abi_version", "fsr_reconstruct_f64",
            "fsr_reconstruct_f32", "fsr_reconstruct_rows_f32", "fsr_reconstruct_rows_f64",
            "fsr_reconstruct_device_f32", "fsr_reconstruct_device_f64", "fsr_iterate_spectra",
            "fsr_quarter_sample_device", "fsr_sq_error_device", "fsr_last_stats", "fsr_spatial_oracle",
            "fsr_pin_host", "fsr_unpin_host"]


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, int):
        return ctypes.c_void_p(a)
    return a.ctypes.data_as(ctypes.c_void_p)


def make_params(block=4, border=14, iterations=100, rho=0.7, gamma=0.5, reducer="tree",
                early_stop=False, precision="fp64", argmax="redux", guard_tau=0.0,
                kernel="auto", guard_kappa=0.0) -> FsrParamsC:
    p = FsrParamsC()
    load().fsr_params_init(ctypes.byref(p))
    if reducer not in REDUCER:
        raise ValueError(f"unknown argmax strategy {reducer!r}, expected one of ('tree', 'linear')")
    if precision not in PRECISION:
        raise ValueError(f"unknown precision {precision!r}, expected one of {tuple(PRECISION)}")
    if argmax not in ARGMAX:
        raise ValueError(f"unknown argmax implementation {argmax!r}, expected one of {tuple(ARGMAX)}")
    p.block, p.border, p.iterations = int(block), int(border), int(iterations)
    p.rho, p.gamma = float(rho), float(gamma)
    p.reducer, p.early_stop = REDUCER[reducer], 1 if early_stop else 0
    if kernel not in KERNEL:
        raise ValueError(f"unknown kernel variant {kernel!r}, expected one of {tuple(KERNEL)}")
    p.precision, p.argmax_impl, p.guard_tau = PRECISION[precision], ARGMAX[argmax], float(guard_tau)
    p.kernel = KERNEL[kernel]
    p.guard_kappa = float(guard_kappa)
    return p


class _OutputPool:
    """Host memory for returned images, recycled once no array references it.

    A fresh 4K f64 output (66 MB) costs ~1.5 ms of first-touch page faults per
    call inside the engine's copy-out; the pool hands out memory that was
    faulted in by an earlier call.  Buffers of PIN_MIN bytes or more are
    anonymous mappings (whole pages of their own) page-locked once with
    fsr_pin_host, so the engine DMAs results straight into them (no staging
    copy-out).  Every call still returns a NEW array (the reference returns a
    fresh GrayImage, core.py:24): its memory goes back to the pool only when
    the array and every view of it are gone (_Lease)."""

    PIN_MIN = 1 << 20

    def __init__(self, max_cached_bytes=1 << 30):
        self._free = {}
        self._cached = 0
        self._max = max_cached_bytes
        self._lock = threading.Lock()

    @staticmethod
    def _addr(buf):
        c = ctypes.c_char.from_buffer(buf)
        a = ctypes.addressof(c)
        del c
        return a

    def take(self, nbytes):
        with self._lock:
            lst = self._free.get(nbytes)
            if lst:
                self._cached -= nbytes
                return lst.pop()
        if nbytes < self.PIN_MIN:
            return bytearray(nbytes)
        buf = mmap.mmap(-1, nbytes)
        try:  # page-locking is an optimisation: on failure the engine stages as usual
            load().fsr_pin_host(self._addr(buf), nbytes)
        except Exception:
            pass
        return buf

    def give_back(self, buf):
        with self._lock:
            if self._cached + len(buf) <= self._max:
                self._free.setdefault(len(buf), []).append(buf)
                self._cached += len(buf)
                return
        if isinstance(buf, mmap.mmap):
            try:
                load().fsr_unpin_host(self._addr(buf))
            except Exception:
                pass
            buf.close()


class _Lease:
    """Buffer exporter of one returned array (PEP 688): numpy keeps it alive
    through the array's base chain, so __del__ runs after the last view dies."""

    __slots__ = ("buf", "pool")

    def __init__(self, buf, pool):
        self.buf = buf
        self.pool = pool

    def __buffer__(self, flags):
        return memoryview(self.buf)

    def __del__(self):
        try:
            self.pool.give_back(self.buf)
        except Exception:  # interpreter shutdown
            pass


_OUT = _OutputPool()


def new_image(shape, dtype):
    """A new, writable, C-contiguous array on recycled host memory."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    return np.frombuffer(_Lease(_OUT.take(n), _OUT), dtype=dt).reshape(shape)


class Engine:
    """One libfsr engine over a set of CUDA devices (strip-partitioned)."""

    def __init__(self, devices=None):
        L = load()
        self._L = L
        h = ctypes.c_void_p()
        if devices:
            arr = (ctypes.c_int32 * len(devices))(*devices)
            rc = L.fsr_engine_create(ctypes.cast(arr, ctypes.c_void_p), len(devices), ctypes.byref(h))
        else:
            rc = L.fsr_engine_create(None, 0, ctypes.byref(h))
        if rc != FSR_OK:
            raise RuntimeError(L.fsr_last_error(None).decode())
        self._h = h
        self.devices = tuple(devices) if devices else (0,)

    def close(self):
        if getattr(self, "_h", None):
            self._L.fsr_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc == FSR_OK:
            return
        msg = self._L.fsr_last_error(self._h).decode()
        if rc in (FSR_EINVAL, FSR_ENOSAMPLES, FSR_EUNSUPPORTED):
            raise ValueError(msg)
        raise RuntimeError(msg)

    def reconstruct(self, px, mask, params: FsrParamsC, sel=None, done=None):
        """Host-buffer whole-image call; returns a new array (never aliases px)."""
        px = np.ascontiguousarray(px)
        if px.dtype not in (np.float32, np.float64):
            px = px.astype(np.float64)
        mask = np.ascontiguousarray(mask, dtype=np.uint8) if mask.dtype != np.bool_ \
            else np.ascontiguousarray(mask).view(np.uint8)
        h, w = px.shape
        out = new_image(px.shape, px.dtype)
        fn = self._L.fsr_reconstruct_f64 if px.dtype == np.float64 else self._L.fsr_reconstruct_f32
        self._check(fn(self._h, ctypes.byref(params), _ptr(px), _ptr(mask), h, w, _ptr(out),
                       _ptr(sel), _ptr(done)))
        return out

    def reconstruct_rows(self, px, mask, params: FsrParamsC, row0: int, row1: int, out,
                         fill: float = float("nan")):
        """Strip call on host buffers: block rows [row0, row1) into ``out`` (full size).
        ``fill``: the empty-support value (the whole frame's mean of the known
        samples); NaN = computed from ``px``/``mask``, which must then hold every row."""
        h, w = px.shape
        assert px.dtype in (np.float32, np.float64) and out.dtype == px.dtype and mask.dtype == np.uint8
        assert px.flags.c_contiguous and out.flags.c_contiguous and mask.flags.c_contiguous
        fn = self._L.fsr_reconstruct_rows_f64 if px.dtype == np.float64 else self._L.fsr_reconstruct_rows_f32
        self._check(fn(self._h, ctypes.byref(params), _ptr(px), _ptr(mask), h, w, row0, row1,
                       float(fill), _ptr(out)))
        return out

    def reconstruct_device(self, d_px, px_pitch, d_mask, mask_pitch, height, width, row0, row1,
                           d_out, out_pitch, params: FsrParamsC, stream=0,
                           fill: float = float("nan"), *, io: str):
        """Device pointers (ints), asynchronous on ``stream`` (a cudaStream_t as int).
        ``io`` (required: raw pointers carry no dtype): pixel type "f32" or "f64"
        of d_px and d_out; ``fill`` as in reconstruct_rows (NaN:
        the device computes the mean from all ``height`` rows of d_px/d_mask)."""
        fn = {"f32": self._L.fsr_reconstruct_device_f32, "f64": self._L.fsr_reconstruct_device_f64}[io]
        self._check(fn(self._h, ctypes.byref(params), ctypes.c_void_p(d_px), px_pitch,
                       ctypes.c_void_p(d_mask), mask_pitch, height, width, row0, row1,
                       ctypes.c_void_p(d_out), out_pitch, float(fill), ctypes.c_void_p(stream)))

    def iterate_spectra(self, R, G, W, wf, params: FsrParamsC, thr=None, sel=None, obj=None,
                        ties=None, done=None):
        """Array-level loop operator, in place on complex128 R and G."""
        for name, a in (("R", R), ("G", G)):
            if a.dtype != np.complex128 or not a.flags.c_contiguous:
                raise ValueError(f"{name} must be C-contiguous complex128")
        count, n, _ = R.shape
        W = np.ascontiguousarray(W, dtype=np.complex128)
        wf = np.ascontiguousarray(wf, dtype=np.float64)
        thr = None if thr is None else np.ascontiguousarray(thr, dtype=np.float64)
        self._check(self._L.fsr_iterate_spectra(
            self._h, ctypes.byref(params), count, n, _ptr(R), _ptr(G), _ptr(W), _ptr(wf),
            _ptr(thr), _ptr(sel), _ptr(obj), _ptr(ties), _ptr(done)))

    def spatial_oracle(self, signal, mask, spatial, wf, gamma: float, iterations: int):
        """FFT-free spatial-domain oracle (oracle.py:25-132) on [count, S, S] blocks:
        returns (out, objectives, selections, ties, energies)."""
        signal = np.ascontiguousarray(signal, dtype=np.float64)
        if signal.ndim != 3 or signal.shape[1] != signal.shape[2]:
            raise ValueError("signal must be [count, S, S]")
        count, S, _ = signal.shape
        mask = np.ascontiguousarray(mask, dtype=np.uint8).reshape(count, S, S)
        spatial = np.ascontiguousarray(spatial, dtype=np.float64).reshape(count, S, S)
        wf = np.ascontiguousarray(wf, dtype=np.float64).reshape(S, S)
        it = int(iterations)
        out = np.empty((count, S, S), np.float64)
        obj = np.empty((count, max(it, 1)), np.float64)
        sel = np.empty((count, max(it, 1)), np.int32)
        ties = np.empty((count, max(it, 1)), np.uint8)
        en = np.empty((count, it + 1), np.float64)
        self._check(self._L.fsr_spatial_oracle(
            self._h, S, it, float(gamma), count, _ptr(signal), _ptr(mask), _ptr(spatial), _ptr(wf),
            _ptr(out), _ptr(obj), _ptr(sel), _ptr(ties), _ptr(en)))
        return out, obj[:, :it], sel[:, :it], ties[:, :it].astype(bool), en

    def quarter_sample_device(self, d_img, img_pitch, height, width, seed, d_sampled, sampled_pitch,
                              d_mask, mask_pitch, stream=0):
        """On-device quarter sampling (sampling.py:53-80), asynchronous on ``stream``."""
        self._check(self._L.fsr_quarter_sample_device(
            self._h, ctypes.c_void_p(d_img), img_pitch, height, width, ctypes.c_uint64(seed & (2**64 - 1)),
            ctypes.c_void_p(d_sampled), sampled_pitch, ctypes.c_void_p(d_mask), mask_pitch,
            ctypes.c_void_p(stream)))

    def sq_error_device(self, d_ref, ref_pitch, d_test, test_pitch, height, width, d_sse, stream=0):
        """*d_sse = sum (clamp(test, 0, 255) - ref)^2 in fp64 (metrics.py:35-48), asynchronous."""
        self._check(self._L.fsr_sq_error_device(
            self._h, ctypes.c_void_p(d_ref), ref_pitch, ctypes.c_void_p(d_test), test_pitch, height,
            width, ctypes.c_void_p(d_sse), ctypes.c_void_p(stream)))

    def last_stats(self) -> dict:
        """Statistics of the last call (waits for an asynchronous device call);
        raises ValueError("no known samples") if that call found an empty window
        in a frame without any known sample."""
        s = FsrStatsC()
        self._check(self._L.fsr_last_stats(self._h, ctypes.byref(s)))
        d = {f: getattr(s, f) for f, _ in FsrStatsC._fields_ if f != "reserved"}
        d["served_fp64"] = bool(s.flags & 2)  # FSR_STATS_SERVED_FP64
        return d


_default = {}
_default_lock = threading.Lock()


def default_engine(devices=None) -> Engine:
    key = tuple(devices) if devices else (0,)
    with _default_lock:
        eng = _default.get(key)
        if eng is None:
            eng = Engine(list(key))
            _default[key] = eng
        return eng
