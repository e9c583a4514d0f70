"""Host-resident batches through the evaluator with copy/compute overlap.

The reference evaluates ciphertexts that live in host memory
(``Polynomial`` rows, poly.hpp:74-119); a drop-in caller hands this package
host ciphertexts and wants host results back.  Doing that naively
(copy everything in, compute, copy everything out) leaves the GPU idle for
the whole PCIe transfer.  ``HostPipeline`` cuts the batch into chunks and
runs three stream-ordered stages per chunk —

    H2D (copy stream)  ->  evaluator calls (compute stream of the slot)  ->  D2H (copy-out stream)

with ``depth`` compute slots, each with its own device input buffers and its
own stream (so its own scratch arena inside the native library).  PCIe is
full duplex, so in steady state chunk k+1 is copied in while chunk k is
evaluated and chunk k-1 is copied out; consecutive ``run`` calls keep the
pipeline full (no host synchronisation between them).

Everything on the compute streams is the normal public API (``ckks.hmult``,
``ckks.hrot`` ...) — this module only schedules copies and streams.
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import torch


class HostPipeline:
    """Chunked H2D -> compute -> D2H over pinned host tensors.

    ``fn(dev_inputs) -> dev_outputs`` is called once per chunk on the slot's
    compute stream; its inputs are device views ``[chunk, ...]`` of the
    host inputs and it returns device tensors whose leading dimension is the
    chunk (copied into the matching rows of the host outputs).
    """

    def __init__(self, device: torch.device, chunk: int, depth: int = 2):
        if chunk < 1 or depth < 1:
            raise ValueError("chunk and depth must be positive")
        self.device = torch.device(device)
        self.chunk, self.depth = chunk, depth
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.comp = [torch.cuda.Stream(self.device) for _ in range(depth)]
        self._bufs: List[List[torch.Tensor]] = [[] for _ in range(depth)]
        self._obufs: List[List[torch.Tensor]] = [[] for _ in range(depth)]
        self._drained = [None] * depth  # event: slot's output buffers copied to the host
        self._freed = [None] * depth   # event: slot's compute finished reading its inputs
        self._slot = 0

    def _slot_outs(self, slot: int, host_out: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        bufs = self._obufs[slot]
        want = [(self.chunk,) + tuple(h.shape[1:]) for h in host_out]
        if len(bufs) != len(host_out) or any(tuple(b.shape) != w or b.dtype != h.dtype
                                             for b, w, h in zip(bufs, want, host_out)):
            bufs = [torch.empty(w, dtype=h.dtype, device=self.device) for w, h in zip(want, host_out)]
            self._obufs[slot] = bufs
        return bufs

    def _slot_bufs(self, slot: int, host_in: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        bufs = self._bufs[slot]
        want = [(self.chunk,) + tuple(h.shape[1:]) for h in host_in]
        if len(bufs) != len(host_in) or any(tuple(b.shape) != w or b.dtype != h.dtype
                                            for b, w, h in zip(bufs, want, host_in)):
            bufs = [torch.empty(w, dtype=h.dtype, device=self.device) for w, h in zip(want, host_in)]
            self._bufs[slot] = bufs
        return bufs

    def run(self, host_in: Sequence[torch.Tensor], fn: Callable[..., Sequence[torch.Tensor]],
            host_out: Sequence[torch.Tensor], outputs_in_place: bool = False) -> torch.cuda.Event:
        """Enqueue the whole batch; returns an event recorded after the last
        D2H (wait on it, or synchronise, before reading ``host_out``).  The
        caller's current stream is NOT made to wait, so back-to-back calls
        overlap; order later work with ``stream.wait_event(returned)``.

        ``outputs_in_place``: ``fn(dev_inputs, dev_outputs)`` writes into
        per-slot device output buffers the pipeline owns (e.g. through the
        evaluator's ``out=`` arguments), so a steady-state step allocates no
        device memory at all."""
        B = host_in[0].shape[0]
        if any(h.shape[0] != B for h in list(host_in) + list(host_out)):
            raise ValueError("host inputs and outputs must share the batch dimension")
        for h in list(host_in) + list(host_out):
            if h.is_cuda or not h.is_pinned():
                raise ValueError("host tensors must be pinned CPU memory")
        cur = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(cur)
        self.h2d.wait_event(start)
        self.d2h.wait_event(start)
        for lo in range(0, B, self.chunk):
            hi = min(B, lo + self.chunk)
            n = hi - lo
            slot = self._slot
            self._slot = (slot + 1) % self.depth
            s = self.comp[slot]
            s.wait_event(start)
            bufs = self._slot_bufs(slot, host_in)
            if self._freed[slot] is not None:
                self.h2d.wait_event(self._freed[slot])
            with torch.cuda.stream(self.h2d):
                for b, h in zip(bufs, host_in):
                    b[:n].copy_(h[lo:hi], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(self.h2d)
            s.wait_event(loaded)
            if outputs_in_place:
                obufs = self._slot_outs(slot, host_out)
                if self._drained[slot] is not None:  # the slot's previous outputs reached the host
                    s.wait_event(self._drained[slot])
            with torch.cuda.stream(s):
                outs = fn([b[:n] for b in bufs], [o[:n] for o in obufs]) if outputs_in_place else \
                    fn([b[:n] for b in bufs])
                done = torch.cuda.Event()
                done.record(s)
            self._freed[slot] = done
            self.d2h.wait_event(done)
            with torch.cuda.stream(self.d2h):
                for o, h in zip(outs, host_out):
                    if not outputs_in_place:
                        o.record_stream(self.d2h)  # allocated on s, read on d2h
                    h[lo:hi].copy_(o, non_blocking=True)
                if outputs_in_place:
                    drained = torch.cuda.Event()
                    drained.record(self.d2h)
                    self._drained[slot] = drained
        end = torch.cuda.Event()
        end.record(self.d2h)
        return end


class CapturedStep:
    """A fixed sequence of evaluator calls captured once in a CUDA graph and
    replayed (small batches / single-ciphertext serving, where the ~1 us
    GPU-side gap between the ~23 kernels of every mechanism is a large share
    of the time: +19% ops/s at B = 1, `profiles/round1_session2.md`).

    ``fn()`` must read its inputs from, and return, tensors that stay alive
    (static buffers): refresh inputs in place (``x.copy_(new)``) between
    replays.  The native library allocates nothing during the capture as
    long as ``fn`` ran once before (its per-stream scratch arena is sized by
    the warm-up), which ``CapturedStep`` does.
    """

    def __init__(self, device: torch.device, fn: Callable[[], object], warmup: int = 2):
        self.device = torch.device(device)
        self.stream = torch.cuda.Stream(self.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            for _ in range(max(1, warmup)):
                fn()
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.outputs = fn()

    def replay(self):
        """Enqueue one replay on the capture stream (ordered after the caller's
        current stream) and make the caller's stream wait for it."""
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        self.graph.replay()
        cur.wait_stream(self.stream)
        return self.outputs
