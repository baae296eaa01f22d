"""Thin ctypes binding of librkc.so (include/rkc.h) -- argument marshalling only.

Every step of the path runs in the CUDA kernels of librkc.so; this module
only converts numpy arrays / torch tensors to pointers.  It fails loudly
(ImportError) when the library is missing: there is no CPU fallback.
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RKC_LIB selects an alternative in-tree build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("RKC_LIB") or os.path.join(_HERE, "librkc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2605_24259_b200/build.py` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---- status codes / constants (include/rkc.h) -----------------------------
RKC_OK, RKC_E_INVAL, RKC_E_NOMEM, RKC_E_CUDA, RKC_E_OVERFLOW, RKC_E_LOST, RKC_E_STATE = \
    0, -1, -2, -3, -4, -5, -6
RKC_NCTR = 32
RKC_NHIST = 128
RKC_HIST_CLAIM, RKC_HIST_REQ, RKC_HIST_CTR = 0, 42, 48

EVENT = np.dtype([("trace", "<u4"), ("step", "<u4"), ("type", "u1"), ("seq", "u1"),
                  ("slot", "u1"), ("reason", "u1"), ("mask", "<u4"), ("f", "<u4", (4,))])
BLOCK_VIEW = np.dtype([("res", "u1"), ("owner", "u1"), ("pad", "<u2"), ("pos", "<u4"),
                       ("seq", "<u4")])
CLAIM_VIEW = np.dtype([("state", "u1"), ("mode", "u1"), ("obj", "u1"), ("pad", "u1"),
                       ("F", "<u4"), ("R", "<u4"), ("D", "<u4"), ("decision_step", "<u4"),
                       ("protected_blocks", "<u4")])
REQUEST_VIEW = np.dtype([("status", "u1"), ("write_admit", "u1"), ("target", "u1"),
                         ("defer_count", "u1"), ("prompt", "<u4"), ("chunk", "<u4"),
                         ("decode", "<u4"), ("done", "<u4"), ("live", "<u4"), ("hit", "<u4"),
                         ("pad", "<u4")])
OBJECT_VIEW = np.dtype([("live", "u1"), ("claim", "u1"), ("pad", "u1", (2,)), ("len", "<u4"),
                        ("leading", "<u4")])
HEADER_VIEW = np.dtype([("seq_ctr", "<u4"), ("free_blocks", "<u4"), ("alive", "<u4"),
                        ("protected_total", "<u4")])
CLAIM_INPUT = np.dtype([("trace", "<u4"), ("claim_slot", "u1"), ("object_slot", "u1"),
                        ("mode", "u1"), ("pad", "u1"), ("footprint_blocks", "<u4"),
                        ("required_leading_blocks", "<u4"), ("duration_steps", "<u4"),
                        ("pad2", "<u4"), ("cache_identity", "<u8"), ("claim_id", "<u8"), ("owner_scope", "<u8")])
REQUEST_INPUT = np.dtype([("trace", "<u4"), ("request_slot", "u1"), ("target_object", "u1"),
                          ("write_admit", "u1"), ("pad", "u1"), ("prompt_tokens", "<u4"),
                          ("chunk_tokens", "<u4"), ("decode_tokens", "<u4"), ("pad2", "<u4"),
                          ("request_id", "<u8")])
TRACE_OP = np.dtype([("trace", "<u4"), ("kind", "u1"), ("a", "u1"), ("b", "u1"), ("c", "u1"),
                     ("x", "<u4"), ("y", "<u4"), ("z", "<u4")])
assert EVENT.itemsize == 32 and CLAIM_INPUT.itemsize == 48 and REQUEST_INPUT.itemsize == 32
assert TRACE_OP.itemsize == 20


class rkc_pool_config(ctypes.Structure):
    _fields_ = [("num_traces", ctypes.c_uint32), ("max_blocks", ctypes.c_uint32),
                ("max_claims", ctypes.c_uint32), ("max_requests", ctypes.c_uint32),
                ("max_objects", ctypes.c_uint32), ("events_per_trace", ctypes.c_uint32),
                ("pool_identity", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


_vp, _u32, _u64, _i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
_sigs = {
    "rkc_abi_version": (ctypes.c_int, []),
    "rkc_status_string": (ctypes.c_char_p, [ctypes.c_int32]),
    "rkc_pool_create": (ctypes.c_int32, [ctypes.POINTER(rkc_pool_config), _vp, ctypes.POINTER(_vp)]),
    "rkc_pool_destroy": (ctypes.c_int32, [_vp]),
    "rkc_pool_reset": (ctypes.c_int32, [_vp, _vp]),
    "rkc_pool_info": (ctypes.c_int32, [_vp, ctypes.POINTER(rkc_pool_config), ctypes.POINTER(_u64),
                                       ctypes.POINTER(_u64)]),
    "rkc_claim_submit": (ctypes.c_int32, [_vp, _vp, _u32, _i32, _vp]),
    "rkc_request_admit": (ctypes.c_int32, [_vp, _vp, _u32, _i32, _vp]),
    "rkc_op_stage": (ctypes.c_int32, [_vp, _vp, _u32, _i32, _vp]),
    "rkc_step_batch": (ctypes.c_int32, [_vp, _vp, _u32, _i32, _vp]),
    "rkc_telemetry_read": (ctypes.c_int32, [_vp, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp, _i32,
                                            _i32, _vp]),
    "rkc_state_export": (ctypes.c_int32, [_vp, _u32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "rkc_state_import": (ctypes.c_int32, [_vp, _u32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "rkc_staging_conflicts": (ctypes.c_int32, [_vp, ctypes.POINTER(_u64)]),
    "rkc_state_set_step": (ctypes.c_int32, [_vp, _u64]),
    "rkc_launch_count": (ctypes.c_ulonglong, []),
    "rkc_conformance_check": (ctypes.c_int32, [_vp, _vp, _u32, _vp, _u32, _vp, _vp, _vp, _vp]),
    "rkc_pool_conformance": (ctypes.c_int32, [_vp, _vp, _vp, _vp]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED_SYMBOLS = tuple(_sigs)


RKC_CHECK = {"L1": 0x01, "L2": 0x02, "L3": 0x04, "L45": 0x08, "L6": 0x10, "L7": 0x20, "I4": 0x40,
             "LOST": 0x80}
RKC_NEVIDENCE = 9
EVIDENCE_NAMES = ["accepted", "materialized", "harmed", "refusals", "attributed_refusals", "victims",
                  "after_release_victims", "write_denials", "failing_traces"]


class RkcError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_lib.rkc_status_string(status).decode()} ({status})")


def _check(status: int, where: str, ok=(RKC_OK,)):
    if status not in ok:
        raise RkcError(status, where)
    return status


def _ptr(x) -> int | None:
    """numpy array / torch tensor / int / None -> raw pointer."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    raise TypeError(type(x))


def _on_device(x) -> int:
    return 1 if (hasattr(x, "is_cuda") and x.is_cuda) else 0


def _count(x, record_size: int) -> int:
    """number of records in a numpy record array or a raw byte tensor"""
    if isinstance(x, np.ndarray) and x.dtype.itemsize == record_size:
        return len(x)
    nbytes = x.nbytes if isinstance(x, np.ndarray) else x.numel() * x.element_size()
    assert nbytes % record_size == 0
    return nbytes // record_size


def _stream(stream, device: int | None = None) -> int | None:
    """A stream handle; None means torch's current stream on `device` (the
    pool's device, so a pool on cuda:k is never driven from another device's
    stream)."""
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream(device).cuda_stream
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def rkc_abi_version() -> int:
    return _lib.rkc_abi_version()


def rkc_launch_count() -> int:
    return int(_lib.rkc_launch_count())


class Pool:
    """One pool of `num_traces` independent paged-KV allocator traces on one GPU.

    Method names follow the C ABI (rkc_pool_create, rkc_claim_submit,
    rkc_request_admit, rkc_step_batch, rkc_telemetry_read, ...)."""

    def __init__(self, trace_cfgs: np.ndarray, max_blocks: int, max_claims: int = 16,
                 max_requests: int = 16, max_objects: int = 64, events_per_trace: int = 256,
                 pool_identity: int = 0, device: int = 0):
        cfgs = np.ascontiguousarray(trace_cfgs)
        assert cfgs.dtype.itemsize == 12
        self.num_traces = len(cfgs)
        self.max_blocks, self.C, self.Q, self.O = max_blocks, max_claims, max_requests, max_objects
        self.events_per_trace = events_per_trace
        self.device = device
        self.cfg = rkc_pool_config(self.num_traces, max_blocks, max_claims, max_requests,
                                   max_objects, events_per_trace, pool_identity, device, 0)
        self._cfgs = cfgs
        h = _vp()
        _check(_lib.rkc_pool_create(ctypes.byref(self.cfg), cfgs.ctypes.data, ctypes.byref(h)),
               "rkc_pool_create")
        self.handle = h

    def _st(self, stream):
        return _stream(stream, self.device)

    # -- lifecycle -----------------------------------------------------------
    def rkc_pool_destroy(self):
        if getattr(self, "handle", None):
            _check(_lib.rkc_pool_destroy(self.handle), "rkc_pool_destroy")
            self.handle = None

    close = rkc_pool_destroy

    def __del__(self):
        try:
            self.rkc_pool_destroy()
        except Exception:
            pass

    def rkc_pool_reset(self, stream=None):
        _check(_lib.rkc_pool_reset(self.handle, self._st(stream)), "rkc_pool_reset")

    def rkc_pool_info(self):
        c = rkc_pool_config()
        step, nbytes = _u64(), _u64()
        _check(_lib.rkc_pool_info(self.handle, ctypes.byref(c), ctypes.byref(step),
                                  ctypes.byref(nbytes)), "rkc_pool_info")
        return dict(step=step.value, device_bytes=nbytes.value, num_traces=c.num_traces)

    # -- staging (online API) ------------------------------------------------
    def rkc_claim_submit(self, claims, stream=None):
        n = _count(claims, CLAIM_INPUT.itemsize)
        return _check(_lib.rkc_claim_submit(self.handle, _ptr(claims), n, _on_device(claims),
                                            self._st(stream)), "rkc_claim_submit")

    def rkc_request_admit(self, reqs, stream=None):
        n = _count(reqs, REQUEST_INPUT.itemsize)
        return _check(_lib.rkc_request_admit(self.handle, _ptr(reqs), n, _on_device(reqs),
                                             self._st(stream)), "rkc_request_admit")

    def rkc_op_stage(self, ops, stream=None):
        n = _count(ops, TRACE_OP.itemsize)
        return _check(_lib.rkc_op_stage(self.handle, _ptr(ops), n, _on_device(ops),
                                        self._st(stream)), "rkc_op_stage")

    def rkc_staging_conflicts(self) -> int:
        v = _u64()
        _check(_lib.rkc_staging_conflicts(self.handle, ctypes.byref(v)), "rkc_staging_conflicts")
        return v.value

    # -- the hot loop --------------------------------------------------------
    def rkc_step_batch(self, ops=None, num_steps: int | None = None, stream=None):
        """ops: None (run the staged step) or [S, num_traces] 16-byte op records
        (numpy host array, or a CUDA uint8/int tensor with S*num_traces*16 bytes)."""
        if ops is None:
            return _check(_lib.rkc_step_batch(self.handle, None, 1, 0, self._st(stream)),
                          "rkc_step_batch")
        if num_steps is None:
            nbytes = ops.nbytes if isinstance(ops, np.ndarray) else ops.numel() * ops.element_size()
            num_steps = nbytes // (16 * self.num_traces)
        return _check(_lib.rkc_step_batch(self.handle, _ptr(ops), int(num_steps), _on_device(ops),
                                          self._st(stream)), "rkc_step_batch")

    # -- telemetry -----------------------------------------------------------
    def rkc_telemetry_read(self, counters_out=None, events_out=None, hist_out=None, drain=False,
                           stream=None, allow_lost=False):
        """Host (numpy) or device (torch) outputs; returns (status, events_written)."""
        outs = [o for o in (counters_out, events_out, hist_out) if o is not None]
        on_dev = 1 if outs and all(_on_device(o) for o in outs) else 0
        if outs and any(_on_device(o) != on_dev for o in outs):
            raise ValueError("mix of host and device outputs")
        cap = 0
        if events_out is not None:
            nbytes = events_out.nbytes if isinstance(events_out, np.ndarray) else \
                events_out.numel() * events_out.element_size()
            cap = nbytes // 32
        written = _u64()
        st = _lib.rkc_telemetry_read(self.handle, _ptr(counters_out), _ptr(events_out), cap,
                                     ctypes.byref(written), _ptr(hist_out), on_dev,
                                     1 if drain else 0, self._st(stream))
        ok = (RKC_OK, RKC_E_LOST) if allow_lost else (RKC_OK,)
        _check(st, "rkc_telemetry_read", ok)
        return st, written.value

    def read_all(self, drain=False):
        """Convenience: (counters[T,32], events[n], hist[128]) as numpy arrays."""
        _, n = self.rkc_telemetry_read()
        counters = np.zeros((self.num_traces, RKC_NCTR), dtype=np.uint32)
        events = np.zeros(n, dtype=EVENT)
        hist = np.zeros(RKC_NHIST, dtype=np.int64)
        self.rkc_telemetry_read(counters, events, hist, drain=drain)
        return counters, events, hist

    # -- test-only views -----------------------------------------------------
    def rkc_state_export(self, trace_begin: int = 0, n: int | None = None):
        n = self.num_traces - trace_begin if n is None else n
        hdr = np.zeros(n, dtype=HEADER_VIEW)
        blocks = np.zeros((n, self.max_blocks), dtype=BLOCK_VIEW)
        claims = np.zeros((n, self.C), dtype=CLAIM_VIEW)
        reqs = np.zeros((n, self.Q), dtype=REQUEST_VIEW)
        objs = np.zeros((n, self.O), dtype=OBJECT_VIEW)
        _check(_lib.rkc_state_export(self.handle, trace_begin, n, hdr.ctypes.data,
                                     blocks.ctypes.data, claims.ctypes.data, reqs.ctypes.data,
                                     objs.ctypes.data), "rkc_state_export")
        return dict(header=hdr, blocks=blocks, claims=claims, requests=reqs, objects=objs)

    def rkc_state_import(self, trace_begin, headers, blocks, claims, reqs, objs):
        n = len(headers)
        arrs = [np.ascontiguousarray(a) for a in (headers, blocks, claims, reqs, objs)]
        _check(_lib.rkc_state_import(self.handle, trace_begin, n, *[a.ctypes.data for a in arrs]),
               "rkc_state_import")

    def rkc_pool_conformance(self, stream=None):
        """Conformance L1-L7 over this pool's event rings; returns (verdict, evidence)
        device tensors."""
        import torch
        verdict = torch.zeros(self.num_traces, dtype=torch.int32, device=f"cuda:{self.device}")
        evidence = torch.zeros(RKC_NEVIDENCE, dtype=torch.int64, device=f"cuda:{self.device}")
        _check(_lib.rkc_pool_conformance(self.handle, _ptr(verdict), _ptr(evidence), self._st(stream)),
               "rkc_pool_conformance")
        return verdict, evidence

    def rkc_state_set_step(self, step: int):
        _check(_lib.rkc_state_set_step(self.handle, step), "rkc_state_set_step")


def rkc_conformance_check(events_dev, offsets_dev, num_traces: int, final_states_dev=None,
                          claims_per_trace: int = 16, lowering_dev=None, stream=None):
    """Conformance L1-L7 over a compacted device event stream; returns
    (verdict[num_traces] u32 tensor, evidence int64[RKC_NEVIDENCE] tensor)."""
    import torch
    dev = events_dev.device
    verdict = torch.zeros(num_traces, dtype=torch.int32, device=dev)
    evidence = torch.zeros(RKC_NEVIDENCE, dtype=torch.int64, device=dev)
    _check(_lib.rkc_conformance_check(_ptr(events_dev), _ptr(offsets_dev), num_traces,
                                      _ptr(final_states_dev), claims_per_trace, _ptr(lowering_dev),
                                      _ptr(verdict), _ptr(evidence), _stream(stream)),
           "rkc_conformance_check")
    return verdict, evidence


def rkc_pool_create(trace_cfgs, max_blocks, **kw) -> Pool:
    return Pool(trace_cfgs, max_blocks, **kw)
