"""Device context: the B200 replacement of the reference's `Simulator` slot.

The reference couples every endpoint to a discrete-event `Simulator`
(`netsim.py:120-204`), which carries the messages of the group allreduce.
Here the transport is device memory: each process owns one arena on its GPU
(send rings, readiness flags, announce words and -- on GPU 0 -- the
activation descriptors), exported to the other processes with CUDA IPC so
kernels read peer send buffers directly over NVLink / NVSwitch. One
`DeviceContext` per process hosts ranks [gpu_index*R, (gpu_index+1)*R).

torch is used for device memory, streams and `torch.distributed` plumbing
(IPC handle exchange); the compute is `libwagma_b200.so`.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from .topology import InvalidParamsError

__all__ = ["DeviceContext", "Job", "JobStatus", "DeviceProtocolFault", "DivergenceError"]


class DeviceProtocolFault(RuntimeError):
    """Device-side protocol violation latched in the arena error word."""

    def __init__(self, code: int, info: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.info = info


class DivergenceError(RuntimeError):
    """Non-finite gradient or loss encountered during training (optim.py:81-82).

    Raised when a fused launch latched WG_EDIVERGE: a rank produced a
    non-finite W' (the reference raises on a non-finite gradient before the
    update, optim.py:174-175). ``rank`` is the first diverging rank.
    """

    def __init__(self, msg: str, rank: int = -1):
        super().__init__(msg)
        self.rank = rank


def _dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return _lib.WG_F32
    if dtype == torch.float64:
        return _lib.WG_F64
    raise InvalidParamsError(f"unsupported dtype {dtype}: float32 or float64")


@dataclass
class Job:
    """One rank's work in one launch (mirrors `wg_job`)."""

    rank: int
    kind: int
    version: int
    W: Optional[torch.Tensor] = None
    m: Optional[torch.Tensor] = None
    g: Optional[torch.Tensor] = None
    fresh: Optional[torch.Tensor] = None
    acc_out: Optional[torch.Tensor] = None
    eta: float = 0.0
    beta: float = 0.0
    momentum: bool = False


@dataclass(frozen=True)
class JobStatus:
    version: int
    contrib_stamp: int
    timely: bool
    activator: bool
    error: int
    root: int = -1  # rank that raised the version's activation flag (-1: none)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class _SlotView:
    """__cuda_array_interface__ wrapper so torch can view a raw device pointer."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        typestr = "<f4" if dtype == torch.float32 else "<f8"
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class DeviceContext:
    """Per-process device state of the WAGMA hot path.

    Parameters mirror the reference's endpoint configuration
    (`GroupAllreduce.__init__`, collective.py:147-159, and
    `OptimizerConfig`, optim.py:106-124): P ranks, group size S, mask rule,
    activation (alpha) versus blocking (beta), staleness bound (tau), plus
    the device-only knobs: send-ring depth, activation grace window and the
    watchdog timeout of every device spin-wait.
    """

    def __init__(self, P: int, S: int, n: int, *, dtype: torch.dtype = torch.float32,
                 tau: Optional[int] = None, mask_rule: str = "example", activation_enabled: bool = True,
                 staleness_bound: Optional[int] = None, ring_depth: int = 0, version_ring: int = 0,
                 grace_us: float = 100.0, timeout_s: float = 20.0, device: Optional[int] = None,
                 n_gpus: int = 1, gpu_index: int = 0, process_group=None):
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceContext needs a CUDA device (B200, sm_100a); there is no CPU path")
        self.lib = _lib.load()
        self.P, self.S, self.n = int(P), int(S), int(n)
        self.dtype = dtype
        self.tau = tau
        # the reference builds every endpoint with staleness_bound=opt.tau
        # (optim.py:386): default to tau, so over-stale contributions fault
        if staleness_bound is None:
            staleness_bound = tau
        self.staleness_bound = int(staleness_bound) if staleness_bound else None
        self.mask_rule = mask_rule
        self.activation_enabled = bool(activation_enabled)
        self.n_gpus, self.gpu_index = int(n_gpus), int(gpu_index)
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.torch_device = torch.device("cuda", self.device)
        if self.P % self.n_gpus:
            raise InvalidParamsError(f"n_gpus={n_gpus} must divide P={P}")
        self.R = self.P // self.n_gpus
        from .dist import rank_layout
        self.local_ranks = rank_layout(self.P, self.n_gpus, self.gpu_index)
        cfg = _lib.WgConfig()
        cfg.P, cfg.S, cfg.n_gpus, cfg.gpu_index, cfg.device = self.P, self.S, self.n_gpus, self.gpu_index, self.device
        cfg.dtype = _dtype_code(dtype)
        cfg.mask_rule = _lib.RULES.get(mask_rule, -1)
        cfg.activation_enabled = 1 if activation_enabled else 0
        cfg.n = self.n
        cfg.tau = int(tau) if tau else 0
        cfg.staleness_bound = int(staleness_bound) if staleness_bound else 0
        cfg.ring_depth = int(ring_depth)
        cfg.version_ring = int(version_ring)
        cfg.grace_ns = int(grace_us * 1000)
        cfg.timeout_ns = int(timeout_s * 1e9)
        self._cfg = cfg
        handle = ctypes.c_void_p()
        torch.cuda.set_device(self.device)
        torch.cuda.init()
        rc = self.lib.wg_ctx_create(ctypes.byref(cfg), ctypes.byref(handle))
        self._raise(rc, "wg_ctx_create")
        self._h = handle
        self._status = _lib.WgJobStatus()
        te, nt, gr, rd = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
        self.lib.wg_ctx_geometry(self._h, ctypes.byref(te), ctypes.byref(nt), ctypes.byref(gr), ctypes.byref(rd))
        self.tile_elems, self.n_tiles, self.grid, self.ring_depth = te.value, nt.value, gr.value, rd.value
        self.launches = 0
        if self.n_gpus > 1:
            self._exchange_handles(process_group)

    # -- errors -----------------------------------------------------------

    def _raise(self, rc: int, what: str) -> None:
        if rc == _lib.WG_OK:
            return
        msg = f"{what}: {self.lib.wg_strerror(rc).decode()} ({_lib.last_error()})"
        if rc == _lib.WG_EINVAL:
            raise InvalidParamsError(msg)
        if rc in (_lib.WG_EVERSION, _lib.WG_ESTALE, _lib.WG_EPROTO, _lib.WG_ESYNC):
            raise DeviceProtocolFault(rc, -1, msg)
        raise RuntimeError(msg)

    def error(self) -> tuple[int, int]:
        code, info = ctypes.c_int(), ctypes.c_int64()
        self._raise(self.lib.wg_ctx_error(self._h, ctypes.byref(code), ctypes.byref(info)), "wg_ctx_error")
        return code.value, info.value

    def _fault(self, code: int, info: int) -> Exception:
        if code == _lib.WG_EDIVERGE:
            return DivergenceError(f"non-finite gradient or replica at rank {info} (device)", rank=info)
        return DeviceProtocolFault(code, info, f"device error {code} "
                                   f"({self.lib.wg_strerror(code).decode()}), info={info}")

    def check(self) -> None:
        """Raise DeviceProtocolFault / DivergenceError if the device latched an error."""
        code, info = self.error()
        if code:
            raise self._fault(code, info)

    def check_async(self) -> None:
        """Like check(), from the host-mapped error mirror: no stream synchronisation.

        Sees the errors of finished launches (and possibly of running ones).
        """
        code, info = ctypes.c_int(), ctypes.c_int64()
        self._raise(self.lib.wg_ctx_error_async(self._h, ctypes.byref(code), ctypes.byref(info)),
                    "wg_ctx_error_async")
        if code.value:
            raise self._fault(code.value, info.value)

    def clear_error(self) -> None:
        self._raise(self.lib.wg_ctx_clear_error(self._h), "wg_ctx_clear_error")

    # -- peers ------------------------------------------------------------

    def export_blob(self) -> bytes:
        buf = ctypes.create_string_buffer(256)
        ln = ctypes.c_size_t(0)
        self._raise(self.lib.wg_ctx_export(self._h, buf, 256, ctypes.byref(ln)), "wg_ctx_export")
        return buf.raw[:ln.value]

    def import_blob(self, gpu_index: int, blob: bytes) -> None:
        self._raise(self.lib.wg_ctx_import_peer(self._h, gpu_index, blob, len(blob)), "wg_ctx_import_peer")

    def _exchange_handles(self, process_group) -> None:
        import torch.distributed as dist

        from .dist import exchange_blobs
        blobs = exchange_blobs(self.gpu_index, self.export_blob(), process_group)
        if sorted(blobs) != list(range(self.n_gpus)):
            raise RuntimeError(f"expected blobs from gpus 0..{self.n_gpus - 1}, got {sorted(blobs)}")
        for gi, blob in blobs.items():
            if gi != self.gpu_index:
                self.import_blob(gi, blob)
        dist.barrier(group=process_group)

    # -- model / send buffers ----------------------------------------------

    def stream_handle(self, stream: Optional[torch.cuda.Stream] = None) -> int:
        s = stream if stream is not None else torch.cuda.current_stream(self.torch_device)
        return s.cuda_stream

    def set_initial_model(self, rank: int, w0: torch.Tensor, stream=None) -> None:
        """SendBuffer(initial_model) with stamp -1 (collective.py:93,169)."""
        self._check_vec(w0, "initial_model")
        self._raise(self.lib.wg_ctx_set_initial_model(self._h, rank, w0.data_ptr(), self.stream_handle(stream)),
                    "wg_ctx_set_initial_model")

    def install(self, rank: int, stamp: int, vec: torch.Tensor, stream=None) -> None:
        """SendBuffer.install outside a fused launch (collective.py:95-101)."""
        self._check_vec(vec, "vec")
        self._raise(self.lib.wg_install(self._h, rank, stamp, vec.data_ptr(), self.stream_handle(stream)),
                    "wg_install")

    def slot(self, rank: int, stamp: int) -> tuple[torch.Tensor, int]:
        """(view of rank's send-ring slot for `stamp`, stamp currently held)."""
        ptr, held = ctypes.c_void_p(), ctypes.c_int64()
        self._raise(self.lib.wg_ctx_slot(self._h, rank, stamp, ctypes.byref(ptr), ctypes.byref(held)),
                    "wg_ctx_slot")
        view = torch.as_tensor(_SlotView(ptr.value, self.n, self.dtype), device=self.torch_device)
        return view, held.value

    def _check_vec(self, t: Optional[torch.Tensor], name: str) -> None:
        if t is None:
            return
        if t.device != self.torch_device or t.dtype != self.dtype or not t.is_contiguous() or t.numel() != self.n:
            raise InvalidParamsError(
                f"{name} must be a contiguous {self.dtype} tensor of {self.n} elements on {self.torch_device}")
        if t.data_ptr() % 16:
            raise InvalidParamsError(f"{name} must be 16-byte aligned")

    # -- launches ---------------------------------------------------------

    def launch(self, jobs: Sequence[Job], forced: Optional[dict[int, Sequence[int]]] = None,
               stream=None) -> None:
        """One fused launch (at most one job per local rank)."""
        arr = (_lib.WgJob * len(jobs))()
        keep = []
        for i, j in enumerate(jobs):
            for name in ("g", "fresh"):  # read-only inputs: realign if needed
                t = getattr(j, name)
                if t is not None and t.data_ptr() % 16:
                    # copy on the launch stream (after the caller's pending work)
                    cur = torch.cuda.current_stream(self.torch_device)
                    ls = stream if stream is not None else cur
                    if ls is not cur:
                        ls.wait_stream(cur)
                    with torch.cuda.stream(ls):
                        t = t.clone()
                    keep.append(t)
                    setattr(j, name, t)
            for name in ("W", "m", "g", "fresh", "acc_out"):
                self._check_vec(getattr(j, name), name)
            a = arr[i]
            a.rank, a.kind, a.version = j.rank, j.kind, j.version
            a.update_rule = _lib.WG_UPDATE_MOMENTUM if j.momentum else _lib.WG_UPDATE_SGD
            a.eta, a.beta = float(j.eta), float(j.beta)
            a.W, a.m, a.g, a.fresh, a.acc_out = _ptr(j.W), _ptr(j.m), _ptr(j.g), _ptr(j.fresh), _ptr(j.acc_out)
        self.launch_array(arr, len(jobs), forced, stream)
        if keep:  # realigned copies must outlive the asynchronous launch
            torch.cuda.current_stream(self.torch_device).synchronize() if stream is None else stream.synchronize()

    def launch_array(self, arr, n_jobs: int, forced: Optional[dict[int, Sequence[int]]] = None, stream=None) -> None:
        """`wg_launch` on a prepared `WgJob` array (the optimizer's fast path;
        the caller has validated every vector it points to)."""
        fv = fs = None
        nf = 0
        if forced:
            nf = len(forced)
            fv = (ctypes.c_int64 * nf)(*forced.keys())
            flat = []
            for v in forced:
                st = list(forced[v])
                if len(st) != self.P:
                    raise InvalidParamsError("forced stamp rows need P entries")
                flat.extend(int(x) for x in st)
            fs = (ctypes.c_int64 * len(flat))(*flat)
        rc = self.lib.wg_launch(self._h, arr, n_jobs, fv, fs, nf, self.stream_handle(stream))
        self._raise(rc, "wg_launch")
        self.launches += 1
        self._n_last = n_jobs

    def statuses(self) -> list[JobStatus]:
        """Per-job status of the last launch (synchronise its stream first)."""
        out = []
        for i in range(self._n_last):
            self._raise(self.lib.wg_launch_status(self._h, i, ctypes.byref(self._status)), "wg_launch_status")
            s = self._status
            out.append(JobStatus(s.version, s.contrib_stamp, bool(s.timely), bool(s.activator), s.error, s.root))
        return out

    def query_version(self, version: int) -> tuple[list[int], bool]:
        """Locked contribution stamps of a group version (device contribution log)."""
        stamps = (ctypes.c_int64 * self.P)()
        locked = ctypes.c_int(0)
        self._raise(self.lib.wg_query_version(self._h, version, stamps, ctypes.byref(locked)), "wg_query_version")
        return list(stamps), bool(locked.value)

    def delay(self, ns: int, stream=None) -> None:
        """Device-side straggler delay on the stream (compute_delay, netsim.py:103-117)."""
        self._raise(self.lib.wg_delay(self._h, int(ns), self.stream_handle(stream)), "wg_delay")

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.wg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def env_rank_info() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))
