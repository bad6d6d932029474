"""Python binding of liblms.so (ctypes over the C ABI in include/lms.h).

This is plumbing: it turns torch tensors and streams into the plain pointers
and handles the C layer takes, and turns negative return codes into the
exception types the reference uses (``ValueError`` family for bad input,
``RuntimeError`` for runtime failures).  There is no fallback: if the
library is missing or CUDA is unavailable, using a :class:`Context` raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblms.so")
SHIM_PATH = os.path.join(_HERE, "liblms_torch.so")   # PyTorch allocator hooks (throw c10 OOM)

LMS_OK, LMS_E_INVALID, LMS_E_OOM, LMS_E_HOST_OOM, LMS_E_CUDA, LMS_E_STATE = 0, -1, -2, -3, -4, -5
CODEC_RAW_CE, CODEC_RAW_SM, CODEC_ZVC, CODEC_ZX = 0, 1, 2, 3
CODECS = {"ce": CODEC_RAW_CE, "sm": CODEC_RAW_SM, "zvc": CODEC_ZVC, "zx": CODEC_ZX}
MAX_DIMS = 8


class LmsError(RuntimeError):
    """A liblms call failed."""


class LmsOutOfMemoryError(LmsError):
    """The enforced device budget cannot satisfy an allocation (SimReport.oom analogue)."""


class _Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("device_reserve", ctypes.c_size_t),
                ("device_limit", ctypes.c_size_t), ("host_reserve", ctypes.c_size_t),
                ("host_chunk", ctypes.c_size_t), ("overlap_transfers", ctypes.c_int),
                ("timing", ctypes.c_int), ("sm_ctas", ctypes.c_int), ("host_limit", ctypes.c_size_t)]


_STAT_FIELDS = [
    "device_in_use", "device_peak", "device_reserved", "device_limit", "device_cached",
    "device_deferred_bytes", "device_mapped", "device_mapped_peak", "n_map", "n_unmap", "n_reclaims", "n_device_syncs",
    "host_in_use", "host_peak", "host_reserved", "n_alloc", "n_free",
    "n_oom", "n_deferred_frees", "n_cross_stream_waits", "n_swap_out", "n_swap_in",
    "n_handles_live", "d2h_logical_bytes", "d2h_wire_bytes", "h2d_logical_bytes",
    "h2d_wire_bytes", "kernel_launches",
]


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in _STAT_FIELDS] + [
        ("d2h_busy_ms", ctypes.c_double), ("h2d_busy_ms", ctypes.c_double),
        ("swap_wait_ms", ctypes.c_double), ("pool_driver_ms", ctypes.c_double),
        ("alloc_wait_ms", ctypes.c_double), ("host_grow_ms", ctypes.c_double),
        ("n_host_grow", ctypes.c_uint64), ("n_scratch_grow", ctypes.c_uint64),
        ("unmap_ms", ctypes.c_double), ("map_ms", ctypes.c_double), ("access_ms", ctypes.c_double),
        ("numa_node", ctypes.c_int64), ("n_host_chunks_on_node", ctypes.c_uint64)]


class _Xfer(ctypes.Structure):
    _fields_ = [("handle_id", ctypes.c_int64), ("direction", ctypes.c_int), ("codec", ctypes.c_int),
                ("logical_bytes", ctypes.c_uint64), ("wire_bytes", ctypes.c_uint64),
                ("start_ms", ctypes.c_double), ("end_ms", ctypes.c_double)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("ready", ctypes.c_int), ("region_bytes", ctypes.c_uint64),
                ("lower_bound_bytes", ctypes.c_uint64), ("n_items", ctypes.c_uint64),
                ("n_planned", ctypes.c_uint64), ("hits", ctypes.c_uint64), ("dynamic", ctypes.c_uint64),
                ("diverged_steps", ctypes.c_uint64), ("solved_bytes", ctypes.c_uint64),
                ("room_bytes", ctypes.c_uint64), ("alpha", ctypes.c_double), ("refinements", ctypes.c_uint64)]


PLAN_OFF, PLAN_RECORD, PLAN_REPLAY, PLAN_REFINE = 0, 1, 2, 3

_lib = None


def lib():
    """Load liblms.so once; raise if it was not built (no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LmsError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                       f"(make -C paper_1807_02037_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    vp, sz, i, i64p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)
    pp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "lms_last_error": ([], ctypes.c_char_p), "lms_version": ([], ctypes.c_char_p),
        "lms_default_config": ([ctypes.POINTER(_Config)], i),
        "lms_create": ([ctypes.POINTER(_Config), pp], i), "lms_destroy": ([vp], i),
        "lms_set_global": ([vp], i), "lms_get_global": ([], vp),
        "lms_set_home_stream": ([vp, vp], i), "lms_set_limit": ([vp, sz], i),
        "lms_reset_peaks": ([vp], i), "lms_get_streams": ([vp, pp, pp], i),
        "lms_set_tuning": ([vp, i, i, i], i),
        "lms_plan_begin": ([vp, i], i), "lms_plan_end": ([vp], i), "lms_plan_reset": ([vp], i),
        "lms_plan_info": ([vp, ctypes.POINTER(_PlanInfo)], i),
        "lms_plan_clock": ([vp, i64p], i),
        "lms_plan_items": ([vp, ctypes.POINTER(ctypes.c_uint64), i64p, i64p, i64p, sz, ctypes.POINTER(sz)], i),
        "lms_plan_solve": ([ctypes.POINTER(ctypes.c_uint64), i64p, i64p, sz, ctypes.POINTER(ctypes.c_uint64),
                            ctypes.POINTER(ctypes.c_uint64)], i),
        "lms_dev_alloc": ([vp, sz, vp, pp], i), "lms_dev_free": ([vp, vp, vp], i),
        "lms_dev_hold_until": ([vp, vp, vp], i), "lms_dev_record_stream": ([vp, vp, vp], i),
        "lms_host_alloc": ([vp, sz, pp], i), "lms_host_free": ([vp, vp], i),
        "lms_host_reserve": ([vp, sz], i),
        "lms_swap_out": ([vp, vp, i64p, i64p, i, i, vp, i, pp], i),
        "lms_swap_in": ([vp, vp, vp, i64p, vp], i), "lms_swap_wait": ([vp, vp, vp], i),
        "lms_swap_out_done": ([vp, vp], i), "lms_handle_release": ([vp, vp], i),
        "lms_handle_info": ([vp, i64p, ctypes.POINTER(ctypes.c_uint64),
                             ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(i)], i),
        "lms_handle_layout": ([vp, i64p, i64p], i),
        "lms_pack": ([vp, vp, vp, i64p, i64p, i, i, vp], i),
        "lms_unpack": ([vp, vp, vp, i64p, i64p, i, i, vp], i),
        "lms_zvc_bound": ([sz], sz), "lms_zvc_encode": ([vp, vp, sz, vp, i, vp], i),
        "lms_zvc_decode": ([vp, vp, sz, vp, vp], i),
        "lms_zvc_encoded_size": ([vp, ctypes.POINTER(sz)], i),
        "lms_stats": ([vp, ctypes.POINTER(_Stats)], i),
        "lms_trace": ([vp, ctypes.POINTER(_Xfer), sz, ctypes.POINTER(sz)], i),
        "lms_trace_clear": ([vp], i), "lms_synchronize": ([vp], i),
        "lms_trim": ([vp, sz, ctypes.POINTER(sz)], i),
        "lms_live_blocks": ([vp, ctypes.POINTER(ctypes.c_uint64), sz, ctypes.POINTER(sz)], i),
        "lms_sim_op": ([vp, pp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), i,
                        pp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), i,
                        ctypes.c_uint64, vp, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc == LMS_OK:
        return
    msg = f"{what}: {lib().lms_last_error().decode()}"
    if rc == LMS_E_INVALID:
        raise ValueError(msg)
    if rc in (LMS_E_OOM, LMS_E_HOST_OOM):
        raise LmsOutOfMemoryError(msg)
    raise LmsError(msg)


def _i64(vals):
    arr = (ctypes.c_int64 * max(1, len(vals)))(*vals)
    return arr


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


@dataclass
class SwapHandle:
    """Host copy of one swapped tensor (opaque ``lms_handle*``)."""

    ptr: int
    id: int
    shape: tuple
    dtype: object
    logical_bytes: int
    restore_strides: tuple
    storage_elems: int
    released: bool = False


class Context:
    """One device's pools and swap channels (``lms_ctx``)."""

    def __init__(self, device: int = 0, device_reserve: int = 0, device_limit: int = 0,
                 host_reserve: int = 0, host_chunk: int = 1 << 30, overlap_transfers: bool = True,
                 timing: bool = False, sm_ctas: int = 0, host_limit: int = 0):
        L = lib()
        cfg = _Config()
        _check(L.lms_default_config(ctypes.byref(cfg)), "lms_default_config")
        cfg.device, cfg.device_reserve, cfg.device_limit = device, device_reserve, device_limit
        cfg.host_reserve, cfg.host_chunk = host_reserve, host_chunk
        cfg.overlap_transfers, cfg.timing, cfg.sm_ctas = int(overlap_transfers), int(timing), sm_ctas
        cfg.host_limit = host_limit
        out = ctypes.c_void_p()
        _check(L.lms_create(ctypes.byref(cfg), ctypes.byref(out)), "lms_create")
        self.ptr = out.value
        self.device = device
        self.timing = timing

    # -- lifetime -------------------------------------------------------------
    def close(self):
        if self.ptr:
            _check(lib().lms_destroy(self.ptr), "lms_destroy")
            self.ptr = None

    def make_global(self):
        _check(lib().lms_set_global(self.ptr), "lms_set_global")

    def set_limit(self, nbytes: int):
        _check(lib().lms_set_limit(self.ptr, nbytes), "lms_set_limit")

    def set_tuning(self, zc_ctas: int = 0, use_bulk: int = -1, use_tma_pack: int = -1):
        """CTAs of the zero-copy kernels (0 = keep), bulk-copy (TMA) use for ZVC and
        tensor-map pack/unpack (-1 = keep)."""
        _check(lib().lms_set_tuning(self.ptr, zc_ctas, use_bulk, use_tma_pack), "lms_set_tuning")

    def reset_peaks(self):
        _check(lib().lms_reset_peaks(self.ptr), "lms_reset_peaks")

    def streams(self):
        """(d2h, h2d) as torch.cuda.ExternalStream objects."""
        import torch
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().lms_get_streams(self.ptr, ctypes.byref(a), ctypes.byref(b)), "lms_get_streams")
        dev = torch.device("cuda", self.device)
        return (torch.cuda.ExternalStream(a.value, device=dev),
                torch.cuda.ExternalStream(b.value, device=dev))

    def _d2h_stream(self):
        s = getattr(self, "_d2h_ext", None)
        if s is None:
            s = self._d2h_ext = self.streams()[0]
        return s

    def trim(self, min_zombies: int = 1) -> int:
        """Unmap stale VA aliases left by page moves once there are at least
        ``min_zombies`` (blocks until the device drains)."""
        n = ctypes.c_size_t()
        _check(lib().lms_trim(self.ptr, min_zombies, ctypes.byref(n)), "lms_trim")
        return n.value

    def synchronize(self):
        _check(lib().lms_synchronize(self.ptr), "lms_synchronize")

    # -- static step plan -------------------------------------------------------
    def plan_begin(self, mode: int):
        """Start a step in PLAN_RECORD or PLAN_REPLAY mode (see include/lms.h)."""
        _check(lib().lms_plan_begin(self.ptr, mode), "lms_plan_begin")

    def plan_end(self):
        """End the step; after a recorded one, place it (LmsOutOfMemoryError: no plan)."""
        _check(lib().lms_plan_end(self.ptr), "lms_plan_end")

    def plan_items(self, cap: int = 1 << 16):
        """The recorded step: (size, alloc event, physical release event, owner's free event)."""
        u64 = (ctypes.c_uint64 * cap)()
        a, b, lg = (ctypes.c_int64 * cap)(), (ctypes.c_int64 * cap)(), (ctypes.c_int64 * cap)()
        n = ctypes.c_size_t()
        _check(lib().lms_plan_items(self.ptr, u64, a, b, lg, cap, ctypes.byref(n)), "lms_plan_items")
        return [(u64[i], a[i], b[i], lg[i]) for i in range(min(cap, n.value))]

    def plan_clock(self) -> int:
        """The recording step's event clock (items' t_alloc/t_free units); -1 outside RECORD."""
        v = ctypes.c_int64()
        _check(lib().lms_plan_clock(self.ptr, ctypes.byref(v)), "lms_plan_clock")
        return v.value

    def plan_reset(self):
        _check(lib().lms_plan_reset(self.ptr), "lms_plan_reset")

    def plan_info(self) -> dict:
        s = _PlanInfo()
        _check(lib().lms_plan_info(self.ptr, ctypes.byref(s)), "lms_plan_info")
        return {f: getattr(s, f) for f, _ in _PlanInfo._fields_}

    # -- swap engine ------------------------------------------------------------
    def swap_out(self, t, codec: str | int = "ce", stream=None) -> SwapHandle:
        """Start moving ``t`` to pinned memory after the work enqueued on ``stream``."""
        code = CODECS[codec] if isinstance(codec, str) else int(codec)
        if not t.is_cuda:
            raise ValueError("swap_out needs a CUDA tensor")
        if t.dim() > MAX_DIMS:
            raise ValueError(f"swap_out supports up to {MAX_DIMS} dims")
        sizes, strides = list(t.shape), list(t.stride())
        h = ctypes.c_void_p()
        _check(lib().lms_swap_out(self.ptr, t.data_ptr(), _i64(sizes), _i64(strides), t.dim(),
                                  t.element_size(), _stream_ptr(stream), code, ctypes.byref(h)),
               "lms_swap_out")
        if _installed is not self and t.numel():
            # liblms holds the source block until the D2H lands only when its own
            # pool owns it (lms.h: lms_swap_out).  Any other allocator (PyTorch's
            # caching allocator when this context is not installed) must not hand
            # the block to the compute stream while the D2H channel still reads it:
            # recordStream defers its reuse past the work now queued on that channel.
            t.record_stream(self._d2h_stream())
        hid = ctypes.c_int64()
        logical = ctypes.c_uint64()
        _check(lib().lms_handle_info(h.value, ctypes.byref(hid), ctypes.byref(logical), None, None),
               "lms_handle_info")
        rs = (ctypes.c_int64 * max(1, t.dim()))()
        se = ctypes.c_int64()
        _check(lib().lms_handle_layout(h.value, rs, ctypes.byref(se)), "lms_handle_layout")
        return SwapHandle(h.value, hid.value, tuple(sizes), t.dtype, logical.value,
                          tuple(rs[k] for k in range(t.dim())), se.value)

    def alloc_for(self, h: SwapHandle):
        """Allocate the swap-in destination in the handle's restore layout."""
        import torch
        return torch.empty_strided(h.shape, h.restore_strides, dtype=h.dtype,
                                   device=torch.device("cuda", self.device))

    def swap_in(self, h: SwapHandle, dst=None, trigger_stream=None):
        """Start the H2D once the work enqueued on ``trigger_stream`` (the control
        op) is done.  Returns the destination tensor; call :meth:`wait` before use."""
        if h.released:
            raise RuntimeError("swap_in of a released handle")
        if dst is None:
            dst = self.alloc_for(h)
        strides = None if tuple(dst.stride()) == h.restore_strides else _i64(list(dst.stride()))
        _check(lib().lms_swap_in(self.ptr, h.ptr, dst.data_ptr(), strides, _stream_ptr(trigger_stream)),
               "lms_swap_in")
        return dst

    def wait(self, h: SwapHandle, stream=None):
        if h.released:
            raise RuntimeError("wait on a released handle")
        _check(lib().lms_swap_wait(self.ptr, h.ptr, _stream_ptr(stream)), "lms_swap_wait")

    def swap_out_done(self, h: SwapHandle) -> bool:
        return lib().lms_swap_out_done(self.ptr, h.ptr) == 1

    def release(self, h: SwapHandle):
        if not h.released:
            h.released = True
            _check(lib().lms_handle_release(self.ptr, h.ptr), "lms_handle_release")

    def handle_codec(self, h: SwapHandle) -> int:
        """The transfer path a swap-out took (CODEC_*; strided views packed in HBM
        and moved by the copy engine report CODEC_RAW_CE)."""
        c = ctypes.c_int()
        _check(lib().lms_handle_info(h.ptr, None, None, None, ctypes.byref(c)), "lms_handle_info")
        return c.value

    def wire_bytes(self, h: SwapHandle) -> int:
        w = ctypes.c_uint64()
        _check(lib().lms_handle_info(h.ptr, None, None, ctypes.byref(w), None), "lms_handle_info")
        return w.value

    # -- pools --------------------------------------------------------------------
    def dev_alloc(self, nbytes: int, stream=None) -> int:
        """Raw device block from this context's pool (for tests / non-torch callers)."""
        p = ctypes.c_void_p()
        _check(lib().lms_dev_alloc(self.ptr, nbytes, _stream_ptr(stream), ctypes.byref(p)), "lms_dev_alloc")
        return p.value

    def dev_free(self, ptr: int, stream=None):
        _check(lib().lms_dev_free(self.ptr, ptr, _stream_ptr(stream)), "lms_dev_free")

    def host_reserve(self, total: int):
        """Grow the pinned pool to ``total`` reserved bytes now (outside timed steps)."""
        _check(lib().lms_host_reserve(self.ptr, total), "lms_host_reserve")

    def hold_until(self, t, stream=None):
        _check(lib().lms_dev_hold_until(self.ptr, t.data_ptr(), _stream_ptr(stream)), "lms_dev_hold_until")

    # -- staging kernels ----------------------------------------------------------
    def pack(self, src, out=None, stream=None):
        """Contiguous copy of a strided view through the sm_100a pack kernels."""
        import torch
        if out is None:
            out = torch.empty(src.shape, dtype=src.dtype, device=src.device)
        _check(lib().lms_pack(self.ptr, out.data_ptr(), src.data_ptr(), _i64(list(src.shape)),
                              _i64(list(src.stride())), src.dim(), src.element_size(), _stream_ptr(stream)),
               "lms_pack")
        return out

    def unpack(self, src, dst, stream=None):
        """Scatter contiguous ``src`` into the strided view ``dst``."""
        _check(lib().lms_unpack(self.ptr, dst.data_ptr(), src.data_ptr(), _i64(list(dst.shape)),
                                _i64(list(dst.stride())), dst.dim(), dst.element_size(), _stream_ptr(stream)),
               "lms_unpack")
        return dst

    def zvc_bound(self, nwords: int) -> int:
        return lib().lms_zvc_bound(nwords)

    def zvc_encode(self, src, dst, stream=None, exponents: bool = False):
        """One-pass encode of ``src``'s 32-bit words into ``dst`` (ZVC v3;
        ``exponents``: the ZX tile forms are allowed too)."""
        _check(lib().lms_zvc_encode(self.ptr, src.data_ptr(), src.numel() * src.element_size() // 4,
                                    dst.data_ptr(), int(exponents), _stream_ptr(stream)), "lms_zvc_encode")

    @staticmethod
    def zvc_encoded_size(enc_host) -> int:
        """Wire bytes of an encoded stream held in host memory (a CPU uint8 tensor)."""
        n = ctypes.c_size_t()
        _check(lib().lms_zvc_encoded_size(enc_host.data_ptr(), ctypes.byref(n)), "lms_zvc_encoded_size")
        return n.value

    def zvc_decode(self, enc, dst, stream=None):
        _check(lib().lms_zvc_decode(self.ptr, enc.data_ptr(), dst.numel() * dst.element_size() // 4,
                                    dst.data_ptr(), _stream_ptr(stream)), "lms_zvc_decode")

    def sim_op(self, outs, ins, errors: int, spin_ns: int = 0, stream=None):
        """One replayed graph op (``lms_sim_op``): ``outs``/``ins`` are lists of
        (device pointer, bytes, pattern tag)."""
        no, ni = len(outs), len(ins)
        P = ctypes.c_void_p * max(1, no)
        Q = ctypes.c_void_p * max(1, ni)
        U64o, U64i = ctypes.c_uint64 * max(1, no), ctypes.c_uint64 * max(1, ni)
        U32o, U32i = ctypes.c_uint32 * max(1, no), ctypes.c_uint32 * max(1, ni)
        _check(lib().lms_sim_op(self.ptr, P(*[o[0] for o in outs]), U64o(*[o[1] for o in outs]),
                                U32o(*[o[2] & 0xFFFFFFFF for o in outs]), no,
                                Q(*[x[0] for x in ins]), U64i(*[x[1] for x in ins]),
                                U32i(*[x[2] & 0xFFFFFFFF for x in ins]), ni, int(spin_ns), errors,
                                _stream_ptr(stream)), "lms_sim_op")

    def swap_out_raw(self, ptr: int, nbytes: int, codec: str | int = "ce", stream=None) -> SwapHandle:
        """Swap out ``nbytes`` of raw device memory (a 1-D byte view)."""
        import torch
        code = CODECS[codec] if isinstance(codec, str) else int(codec)
        h = ctypes.c_void_p()
        _check(lib().lms_swap_out(self.ptr, ptr, _i64([nbytes]), _i64([1]), 1, 1, _stream_ptr(stream), code,
                                  ctypes.byref(h)), "lms_swap_out")
        hid = ctypes.c_int64()
        _check(lib().lms_handle_info(h.value, ctypes.byref(hid), None, None, None), "lms_handle_info")
        return SwapHandle(h.value, hid.value, (nbytes,), torch.uint8, nbytes, (1,), nbytes)

    def swap_in_raw(self, h: SwapHandle, dst_ptr: int, trigger_stream=None):
        if h.released:
            raise RuntimeError("swap_in of a released handle")
        _check(lib().lms_swap_in(self.ptr, h.ptr, dst_ptr, None, _stream_ptr(trigger_stream)), "lms_swap_in")

    # -- reporting ----------------------------------------------------------------
    def stats(self) -> dict:
        s = _Stats()
        _check(lib().lms_stats(self.ptr, ctypes.byref(s)), "lms_stats")
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def trace(self, cap: int = 1 << 16) -> list[dict]:
        buf = (_Xfer * cap)()
        n = ctypes.c_size_t()
        _check(lib().lms_trace(self.ptr, buf, cap, ctypes.byref(n)), "lms_trace")
        return [{f: getattr(buf[k], f) for f, _ in _Xfer._fields_} for k in range(n.value)]

    def live_blocks(self, cap: int = 64) -> tuple[int, list[int]]:
        """(number of live device blocks, sizes of the largest ``cap``)."""
        buf = (ctypes.c_uint64 * cap)()
        n = ctypes.c_size_t()
        _check(lib().lms_live_blocks(self.ptr, buf, cap, ctypes.byref(n)), "lms_live_blocks")
        return n.value, [buf[i] for i in range(min(cap, n.value))]

    def trace_clear(self):
        _check(lib().lms_trace_clear(self.ptr), "lms_trace_clear")


def plan_solve(sizes, t_alloc, t_free):
    """Host-only placement (step_plan.h): offsets (None = not planned) and region size."""
    n = len(sizes)
    u64 = ctypes.c_uint64 * max(1, n)
    offs = u64()
    region = ctypes.c_uint64()
    _check(lib().lms_plan_solve(u64(*sizes), _i64(list(t_alloc)), _i64(list(t_free)), n, offs,
                                ctypes.byref(region)), "lms_plan_solve")
    return [None if offs[i] == 2 ** 64 - 1 else offs[i] for i in range(n)], region.value


class DeviceBuffer:
    """A raw pool block seen as a CUDA array (``__cuda_array_interface__``), so
    ``torch.as_tensor(buf, device="cuda")`` views it without a copy."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3,
                "stream": None}


_installed: Context | None = None


def install_allocator(ctx: Context):
    """Route every PyTorch CUDA allocation of this process through ``ctx``'s pool.

    Must run before the first CUDA allocation (PyTorch's rule for
    ``change_current_allocator``).  Idempotent for the same context.
    """
    global _installed
    import torch
    if _installed is ctx:
        return
    if _installed is not None:
        raise RuntimeError("a different LMS context already owns the PyTorch allocator")
    ctx.make_global()
    if not os.path.exists(SHIM_PATH):
        raise LmsError(f"{SHIM_PATH} is missing; run __graft_entry__.build()")
    alloc = torch.cuda.memory.CUDAPluggableAllocator(SHIM_PATH, "lms_torch_alloc", "lms_torch_free")
    torch.cuda.memory.change_current_allocator(alloc)
    # Tensor.record_stream on our blocks: reuse waits for the recorded streams
    if ctypes.CDLL(SHIM_PATH).lms_torch_hook_record_stream() != 0:
        raise LmsError("could not hook record_stream on the pluggable allocator")
    _installed = ctx


def installed_context() -> Context | None:
    return _installed
