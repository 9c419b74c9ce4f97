"""Thin host-side helpers over the fy_* C ABI for tests and the bench.

torch is used only as plumbing (device allocation, streams, events); every
number is computed by the CUDA kernels in ``lib/liboffsim.so.0``. The
argument meaning and error behaviour are those of ``include/fuyou/fy_adam.h``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from ._lib import (LIB, AdamCounter, AdamHparams, AdamwArgs, Chunk, ChunkTiming, FY_BF16, FY_FP16, FY_FP32,
                   FY_GATHER_NCCL, FY_GATHER_NONE, FY_GATHER_PEER, FY_IPC_HANDLE_BYTES, FY_NCCL_ID_BYTES,
                   FY_SWAP_CPU, FY_SWAP_SSD, FY_TIER_DEVICE, FY_TIER_HOST, PipelineConfig, ShardConfig,
                   ShardIo, ShardSlice, ShardStats, SwapConfig, FyError, check)

_DT = {torch.bfloat16: FY_BF16, torch.float16: FY_FP16, torch.float32: FY_FP32}


def fy_dtype(t: torch.dtype) -> int:
    return _DT[t]


@dataclass
class Hparams:
    """DeepSpeed-0.9.3-CPU-Adam hyper-parameters (see oracle/adamw_oracle.c)."""
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    step: int = 10
    adamw_mode: bool = True
    bias_correction: bool = True
    grad_scale: float = 1.0
    # beta^t given (DeepSpeed running product, from a StepCounter) or None:
    # float(pow(double(beta), step))
    beta_t: Optional[tuple] = None

    def c(self) -> AdamHparams:
        bt = self.beta_t
        return AdamHparams(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                           self.step, int(self.adamw_mode), int(self.bias_correction),
                           self.grad_scale, int(bt is not None), bt[0] if bt else 0.0,
                           bt[1] if bt else 0.0)


class StepCounter:
    """fy_adam_counter: DeepSpeed's Adam_Optimizer step bookkeeping. next(hp)
    returns a copy of hp with beta_t set (one call per chunk update)."""

    def __init__(self, beta1: Optional[float] = None, beta2: Optional[float] = None):
        self.c = AdamCounter()
        if beta1 is not None:
            check(LIB.fy_adam_counter_init(C.byref(self.c), beta1, beta2))

    def next(self, hp: "Hparams") -> "Hparams":
        h = hp.c()
        check(LIB.fy_adam_counter_next(C.byref(self.c), C.byref(h)))
        return dataclasses.replace(hp, beta_t=(h.beta1_t, h.beta2_t))


def workspace_floats() -> int:
    return int(LIB.fy_adamw_workspace_floats())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def adamw_chunk(master: torch.Tensor, exp_avg: torch.Tensor, exp_avg_sq: torch.Tensor,
                grad: torch.Tensor, hp: Hparams, param_out: Optional[torch.Tensor] = None,
                grad_sq_sum: Optional[torch.Tensor] = None, accumulate_sq: bool = False,
                workspace: Optional[torch.Tensor] = None, nonfinite: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None, n: Optional[int] = None,
                grad_scale_dev: Optional[torch.Tensor] = None,
                skip_if_set: Optional[torch.Tensor] = None, lib=None) -> None:
    """Enqueue the fused step on ``stream`` (default: torch's current stream).
    grad_scale_dev (device float32[1]) / skip_if_set (device int32[1]):
    the device-side controls written by clip_coef(). lib: another build of
    the same ABI (the sweep build in kernel sweeps); default the product."""
    if stream is None:
        stream = torch.cuda.current_stream(master.device)
    a = AdamwArgs()
    a.master, a.exp_avg, a.exp_avg_sq = master.data_ptr(), exp_avg.data_ptr(), exp_avg_sq.data_ptr()
    a.grad = grad.data_ptr()
    a.grad_dtype = fy_dtype(grad.dtype)
    a.param_out = _ptr(param_out)
    a.param_dtype = fy_dtype(param_out.dtype) if param_out is not None else FY_BF16
    a.n = master.numel() if n is None else n
    a.hp = hp.c()
    a.grad_sq_sum = _ptr(grad_sq_sum)
    a.accumulate_sq = int(accumulate_sq)
    a.workspace = _ptr(workspace)
    a.nonfinite_flag = _ptr(nonfinite)
    a.grad_scale_dev = _ptr(grad_scale_dev)
    a.skip_if_set = _ptr(skip_if_set)
    lib = LIB if lib is None else lib
    st = lib.fy_adamw_chunk(C.byref(a), C.c_void_p(stream.cuda_stream))
    if st:
        raise FyError(st, lib.fy_last_error().decode())


def clip_coef(grad_sq_sum: torch.Tensor, nonfinite: Optional[torch.Tensor], max_norm: float,
              scale_out: torch.Tensor, skip_out: torch.Tensor,
              stream: Optional[torch.cuda.Stream] = None) -> None:
    """fy_clip_coef: device-side clipping coefficient + overflow skip flag."""
    if stream is None:
        stream = torch.cuda.current_stream(grad_sq_sum.device)
    check(LIB.fy_clip_coef(C.c_void_p(grad_sq_sum.data_ptr()), C.c_void_p(_ptr(nonfinite)),
                           float(max_norm), C.c_void_p(scale_out.data_ptr()),
                           C.c_void_p(skip_out.data_ptr()), C.c_void_p(stream.cuda_stream)))


def adamw_chunks(chunks, hp: Hparams, grad_sq_sum: Optional[torch.Tensor] = None,
                 accumulate_sq: bool = False, workspace: Optional[torch.Tensor] = None,
                 nonfinite: Optional[torch.Tensor] = None,
                 stream: Optional[torch.cuda.Stream] = None,
                 grad_scale_dev: Optional[torch.Tensor] = None,
                 skip_if_set: Optional[torch.Tensor] = None) -> None:
    """fy_adamw_chunks: one multi-chunk launch. ``chunks`` = sequence of
    (master, exp_avg, exp_avg_sq, grad, param_out_or_None)."""
    if stream is None:
        stream = torch.cuda.current_stream(chunks[0][0].device)
    arr = (AdamwArgs * len(chunks))()
    for i, (ms, m, v, g, po) in enumerate(chunks):
        a = arr[i]
        a.master, a.exp_avg, a.exp_avg_sq = ms.data_ptr(), m.data_ptr(), v.data_ptr()
        a.grad = g.data_ptr()
        a.grad_dtype = fy_dtype(g.dtype)
        a.param_out = _ptr(po)
        a.param_dtype = fy_dtype(po.dtype) if po is not None else FY_BF16
        a.n = ms.numel()
        a.hp = hp.c()
        a.grad_sq_sum = _ptr(grad_sq_sum)
        a.accumulate_sq = int(accumulate_sq)
        a.workspace = _ptr(workspace)
        a.nonfinite_flag = _ptr(nonfinite)
        a.grad_scale_dev = _ptr(grad_scale_dev)
        a.skip_if_set = _ptr(skip_if_set)
    check(LIB.fy_adamw_chunks(arr, len(chunks), C.c_void_p(stream.cuda_stream)))


def adamw_chunk_gather(master: torch.Tensor, exp_avg: torch.Tensor, exp_avg_sq: torch.Tensor,
                       grad: torch.Tensor, hp: Hparams, param_out: torch.Tensor, dst_ptrs,
                       grad_sq_sum: Optional[torch.Tensor] = None,
                       workspace: Optional[torch.Tensor] = None,
                       stream: Optional[torch.cuda.Stream] = None, n: Optional[int] = None) -> None:
    """fy_adamw_chunk_gather: the step plus a fused all-gather epilogue that
    stores the updated 16-bit params at every address in ``dst_ptrs`` (where
    this rank's slice starts in each rank's full-param buffer)."""
    if stream is None:
        stream = torch.cuda.current_stream(master.device)
    a = AdamwArgs()
    a.master, a.exp_avg, a.exp_avg_sq = master.data_ptr(), exp_avg.data_ptr(), exp_avg_sq.data_ptr()
    a.grad = grad.data_ptr()
    a.grad_dtype = fy_dtype(grad.dtype)
    a.param_out = param_out.data_ptr()
    a.param_dtype = fy_dtype(param_out.dtype)
    a.n = master.numel() if n is None else n
    a.hp = hp.c()
    a.grad_sq_sum = _ptr(grad_sq_sum)
    a.workspace = _ptr(workspace)
    arr = (C.c_void_p * len(dst_ptrs))(*dst_ptrs)
    check(LIB.fy_adamw_chunk_gather(C.byref(a), arr, len(dst_ptrs), C.c_void_p(stream.cuda_stream)))


def grad_stats(grad: torch.Tensor, grad_scale: float, grad_sq_sum: torch.Tensor,
               workspace: torch.Tensor, nonfinite: Optional[torch.Tensor] = None,
               accumulate: bool = False, stream: Optional[torch.cuda.Stream] = None) -> None:
    if stream is None:
        stream = torch.cuda.current_stream(grad.device)
    check(LIB.fy_grad_stats(C.c_void_p(grad.data_ptr()), fy_dtype(grad.dtype), grad.numel(),
                            grad_scale, C.c_void_p(grad_sq_sum.data_ptr()), int(accumulate),
                            C.c_void_p(workspace.data_ptr()), C.c_void_p(_ptr(nonfinite)),
                            C.c_void_p(stream.cuda_stream)))


def device_info(device: int = 0):
    sm, cps, thr = C.c_int(), C.c_int(), C.c_int()
    check(LIB.fy_device_info(device, C.byref(sm), C.byref(cps), C.byref(thr)))
    return sm.value, cps.value, thr.value


def shard_range(n: int, world: int, rank: int, align: int = 8):
    off, cnt = C.c_uint64(), C.c_uint64()
    check(LIB.fy_shard_range(n, world, rank, align, C.byref(off), C.byref(cnt)))
    return off.value, cnt.value


class ChunkPipeline:
    """Streamed optimizer step over host-resident states (fy_pipeline_*)."""

    def __init__(self, max_chunk_elems: int, slots: int = 3, device: int = 0,
                 grad_dtype: torch.dtype = torch.bfloat16, param_dtype: torch.dtype = torch.bfloat16,
                 grads_on_host: bool = False, params_to_host: bool = True,
                 keep_params_on_device: bool = False, states_on_device: bool = False,
                 no_step_counter: bool = False):
        cfg = PipelineConfig(device, max_chunk_elems, slots, fy_dtype(grad_dtype),
                             fy_dtype(param_dtype), int(grads_on_host), int(params_to_host),
                             int(keep_params_on_device), int(states_on_device), int(no_step_counter))
        h = C.c_void_p()
        check(LIB.fy_pipeline_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._chunks = None

    def close(self):
        if self._h:
            LIB.fy_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, chunks: Sequence[dict], hp: Hparams, want_grad_norm: bool = False) -> None:
        arr = (Chunk * len(chunks))()
        for i, c in enumerate(chunks):
            arr[i] = Chunk(c["n"], c["h_states"], c["grad"], c.get("h_param"), c.get("d_param"),
                           c.get("grad_ready"), c.get("states_stride", 0), c.get("update_done"),
                           c.get("flags", 0))
        self._chunks = arr  # keep alive until wait()
        check(LIB.fy_pipeline_step(self._h, arr, len(chunks), C.byref(hp.c()), int(want_grad_norm)))

    def set_controls(self, grad_scale_dev: Optional[torch.Tensor] = None,
                     skip_if_set: Optional[torch.Tensor] = None) -> None:
        """fy_pipeline_set_controls: device-side clip coefficient / skip flag."""
        check(LIB.fy_pipeline_set_controls(self._h, C.c_void_p(_ptr(grad_scale_dev)),
                                           C.c_void_p(_ptr(skip_if_set))))

    def wait(self):
        sq, bad = C.c_double(), C.c_int()
        check(LIB.fy_pipeline_wait(self._h, C.byref(sq), C.byref(bad)))
        self._chunks = None
        return sq.value, bad.value

    def timings(self, count: int):
        arr = (ChunkTiming * count)()
        total = C.c_uint64()
        check(LIB.fy_pipeline_timings(self._h, arr, count, C.byref(total)))
        return [dict(h2d=(t.h2d_start_ns, t.h2d_end_ns), upd=(t.upd_start_ns, t.upd_end_ns),
                     d2h=(t.d2h_start_ns, t.d2h_end_ns)) for t in arr], total.value


class Swapper:
    """Activation swap engine (fy_swapper_*): GPU -> pinned host (-> SSD)."""
    CPU, SSD = FY_SWAP_CPU, FY_SWAP_SSD

    def __init__(self, device: int = 0, slot_bytes: int = 0, slots: int = 0,
                 file_dir: str = "/tmp", direct_io: bool = True):
        self._dir = file_dir.encode()
        cfg = SwapConfig(device, slot_bytes, slots, self._dir, int(direct_io))
        h = C.c_void_p()
        check(LIB.fy_swapper_create(C.byref(cfg), C.byref(h)))
        self._h = h

    @staticmethod
    def _ev(e):
        return None if e is None else e.cuda_event

    @staticmethod
    def _now(dev):
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream(dev))
        return e

    def swap_out(self, t: torch.Tensor, placement: int, ready=None, src_free=None) -> int:
        """Default `ready`: everything already queued on torch's current
        stream (so a tensor just produced there is complete)."""
        if ready is None:
            ready = self._now(t.device)
        h = C.c_uint64()
        check(LIB.fy_swap_out(self._h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                              placement, self._ev(ready), self._ev(src_free), C.byref(h)))
        return h.value

    def swap_in(self, handle: int, t: torch.Tensor, ready=None, done=None) -> None:
        """Default `ready`: torch's current stream so far; default `done`:
        torch's current stream waits for the restored data (stream-ordered
        like a copy_ on it). Pass events to overlap instead."""
        if ready is None:
            ready = self._now(t.device)
        wait_here = done is None
        if wait_here:
            done = torch.cuda.Event()
            done.record(torch.cuda.current_stream(t.device))  # create it
        check(LIB.fy_swap_in(self._h, handle, C.c_void_p(t.data_ptr()), self._ev(ready), self._ev(done)))
        if wait_here:
            torch.cuda.current_stream(t.device).wait_event(done)

    def release(self, handle: int) -> None:
        check(LIB.fy_swap_release(self._h, handle))

    def sync(self) -> None:
        check(LIB.fy_swapper_sync(self._h))

    def stats(self):
        hb, fb, eng = C.c_uint64(), C.c_uint64(), C.c_char_p()
        check(LIB.fy_swapper_stats(self._h, C.byref(hb), C.byref(fb), C.byref(eng)))
        return dict(host_bytes=hb.value, file_bytes=fb.value, io_engine=eng.value.decode())

    def close(self):
        if self._h:
            LIB.fy_swapper_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """fy_nccl_unique_id: rank 0 creates it, every rank passes the same bytes."""
    buf = C.create_string_buffer(FY_NCCL_ID_BYTES)
    check(LIB.fy_nccl_unique_id(buf))
    return buf.raw


class Shard:
    """Sharded optimizer step across the GPUs of a node (fy_shard_*).

    chunk_elems: every chunk's full size (same on all ranks). gather: "nccl",
    "peer" or None (world 1). tier: "device" (states in HBM) or "host"
    (pinned host states streamed through the chunk pipeline)."""
    GATHER = {None: FY_GATHER_NONE, "none": FY_GATHER_NONE, "nccl": FY_GATHER_NCCL, "peer": FY_GATHER_PEER}

    def __init__(self, chunk_elems: Sequence[int], world: int = 1, rank: int = 0, device: int = 0,
                 gather: Optional[str] = None, nccl_id: Optional[bytes] = None, tier: str = "device",
                 grad_dtype: torch.dtype = torch.bfloat16, param_dtype: torch.dtype = torch.bfloat16,
                 slots: int = 0, piece_elems: int = 0, params_to_host: bool = False,
                 no_step_counter: bool = False, grads_on_host: bool = False):
        self.chunk_elems = list(chunk_elems)
        self._elems = (C.c_uint64 * len(self.chunk_elems))(*self.chunk_elems)
        self._id = C.create_string_buffer(nccl_id, FY_NCCL_ID_BYTES) if nccl_id is not None else None
        cfg = ShardConfig(device, world, rank, self.GATHER[gather],
                          C.cast(self._id, C.c_void_p) if self._id is not None else None,
                          FY_TIER_HOST if tier == "host" else FY_TIER_DEVICE, len(self.chunk_elems),
                          self._elems, fy_dtype(grad_dtype), fy_dtype(param_dtype), slots, piece_elems,
                          int(params_to_host), int(no_step_counter), int(grads_on_host))
        h = C.c_void_p()
        check(LIB.fy_shard_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._io = None
        self._param_dtype, self._device = param_dtype, device
        self.world, self.rank = world, rank

    def slice(self, c: int) -> dict:
        s = ShardSlice()
        check(LIB.fy_shard_slice_info(self._h, c, C.byref(s)))
        return dict(offset=s.offset, count=s.count, stride=s.stride, params=s.params)

    def own_params(self, c: int) -> torch.Tensor:
        """This rank's slot of chunk c's full params in the arena (16-bit,
        `count` elements): the in-place buffer of the reference's convention
        (the update writes the params into the grad buffer,
        proj/src/task_graph.cpp:493-495). A caller that lands the slice's
        gradients here (io grad = this tensor, grad_dtype 16-bit) needs no
        separate gradient memory: 2 B/param of HBM saved."""
        s = self.slice(c)
        dt = self._param_dtype
        if s["count"] == 0:
            return torch.empty(0, dtype=dt, device=torch.device("cuda", self._device))
        ptr = s["params"] + self.rank * s["stride"] * 2
        cai = type("CAI", (), {"__cuda_array_interface__": dict(
            shape=(s["count"],), typestr="<i2", data=(ptr, False), version=3)})()
        return torch.as_tensor(cai, device=torch.device("cuda", self._device)).view(dt)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(FY_IPC_HANDLE_BYTES)
        check(LIB.fy_shard_ipc_handle(self._h, buf))
        return buf.raw

    def connect(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        check(LIB.fy_shard_connect(self._h, C.create_string_buffer(blob, len(blob))))

    def connect_ptrs(self, arenas: Sequence[int]) -> None:
        arr = (C.c_void_p * len(arenas))(*arenas)
        check(LIB.fy_shard_connect_ptrs(self._h, arr))

    def arena(self) -> int:
        """Base of this shard's arena (what peers in the same process pass to
        connect_ptrs)."""
        base, size = C.c_void_p(), C.c_uint64()
        check(LIB.fy_shard_arena(self._h, C.byref(base), C.byref(size)))
        return base.value

    def step(self, io: Sequence[dict], hp: Hparams, want_grad_norm: bool = False,
             stream: Optional[torch.cuda.Stream] = None) -> None:
        """io[c] = dict(states=ptr, grad=ptr[, h_param=ptr, grad_ready=cudaEvent])."""
        arr = (ShardIo * len(io))()
        for i, d in enumerate(io):
            ev = d.get("grad_ready")
            arr[i] = ShardIo(d.get("states"), d.get("grad"), d.get("h_param"),
                             ev.cuda_event if ev is not None and hasattr(ev, "cuda_event") else ev)
        self._io = arr
        if stream is None:
            stream = torch.cuda.current_stream()
        check(LIB.fy_shard_step(self._h, arr, C.byref(hp.c()), int(want_grad_norm),
                                C.c_void_p(stream.cuda_stream)))

    def wait(self):
        sq, bad = C.c_double(), C.c_int()
        check(LIB.fy_shard_wait(self._h, C.byref(sq), C.byref(bad)))
        self._io = None
        return sq.value, bad.value

    def update_ms(self) -> list:
        """Per chunk: device time of its update kernel(s) in the last step."""
        arr = (C.c_double * len(self.chunk_elems))()
        check(LIB.fy_shard_update_ms(self._h, arr, len(self.chunk_elems)))
        return list(arr)

    def stats(self) -> dict:
        st = ShardStats()
        check(LIB.fy_shard_get_stats(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in ShardStats._fields_}

    def close(self):
        if self._h:
            LIB.fy_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
