"""Thin host-side helpers over the fy_* C ABI for tests and the bench.

torch is used only as plumbing (device allocation, streams, events); every
number is computed by the CUDA kernels in ``lib/liboffsim.so.0``. The
argument meaning and error behaviour are those of ``include/fuyou/fy_adam.h``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from ._lib import (LIB, AdamHparams, AdamwArgs, Chunk, ChunkTiming, FY_BF16, FY_FP16, FY_FP32,
                   FY_SWAP_CPU, FY_SWAP_SSD, PipelineConfig, SwapConfig, check)

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

    def c(self) -> AdamHparams:
        return AdamHparams(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                           self.step, int(self.adamw_mode), int(self.bias_correction),
                           self.grad_scale)


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
                skip_if_set: Optional[torch.Tensor] = None) -> None:
    """Enqueue the fused step on ``stream`` (default: torch's current stream).
    grad_scale_dev (device float32[1]) / skip_if_set (device int32[1]):
    the device-side controls written by clip_coef()."""
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
    check(LIB.fy_adamw_chunk(C.byref(a), C.c_void_p(stream.cuda_stream)))


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
                 keep_params_on_device: bool = False, states_on_device: bool = False):
        cfg = PipelineConfig(device, max_chunk_elems, slots, fy_dtype(grad_dtype),
                             fy_dtype(param_dtype), int(grads_on_host), int(params_to_host),
                             int(keep_params_on_device), int(states_on_device))
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
