"""Limb-sharded key switching for one ciphertext over several GPUs
(BASELINE config 4).

The reference evaluates one ciphertext on one host (``key_switch``
ckks.cpp:778-787, ``hmult`` ckks.cpp:804-865, ``hrot`` ckks.cpp:869-897,
``rescale`` ckks.cpp:789-802).  Here the RNS limbs of the ciphertext, of the
ModUp extension and of the key are split across ``world`` ranks: rank s owns
a balanced contiguous block of the Q primes and of the P primes
(:class:`ShardLayout`).  Everything is limb-local except base conversion,
which needs every source row; so each mechanism is

    phase 1 (local)  INTT + BConv part 1 of the owned source rows -> send
    exchange         all-gather of the send buffers (NCCL over NVLink)
    phase 2 (local)  BConv to the owned rows, NTT, KeyMult / combine

once for ModUp (sources: the digit rows) and once for ModDown / rescale
(sources: the P rows and/or the dropped Q rows).  The compute phases are the
C-ABI entry points ``ck_shard_*`` (include/ck32_b200.h); the exchange is a
pluggable object: :class:`TorchExchange` (one rank per process,
``torch.distributed`` all-gather — NCCL on GPUs, gloo in the CPU tests),
:class:`LocalExchange` (several shards driven from one process, used to check
the sharded path against the single-device one on one GPU), or the
peer-memory exchanges :class:`IpcPeerExchange` (one rank per process, buffers
mapped with CUDA IPC) and :class:`LocalPeerExchange` (shards of one process):
there is no gather at all -- phase 1 leaves the INTT rows in the rank's own
exchange buffer and raises a flag in every peer, phase 2 waits for the flags
and its BConv loads the rows straight from the peers' buffers over NVLink
("peer-mapped loads inside BConv").

Outputs are bit-identical to the single-device mechanisms on the owned rows:
the partition does not change any arithmetic.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

MOD_DOWN, RESCALE, MERGED = 0, 1, 2


# ------------------------------------------------------------------ layout --
@dataclass(frozen=True)
class ShardLayout:
    """Row ownership of rank ``rank`` of ``world`` (same partition as the
    native ``Shard``, csrc/ck_context.cu): Q primes [q_lo, q_hi), P primes
    L + [p_lo, p_hi), blocks of sizes floor/ceil(L/world), floor/ceil(alpha/world)."""
    L: int
    alpha: int
    world: int
    rank: int

    @staticmethod
    def _lo(t: int, total: int, world: int) -> int:
        return t * total // world

    def q_block(self, t: Optional[int] = None):
        t = self.rank if t is None else t
        return self._lo(t, self.L, self.world), self._lo(t + 1, self.L, self.world)

    def p_block(self, t: Optional[int] = None):
        t = self.rank if t is None else t
        return self._lo(t, self.alpha, self.world), self._lo(t + 1, self.alpha, self.world)

    @property
    def q_lo(self):
        return self.q_block()[0]

    @property
    def q_hi(self):
        return self.q_block()[1]

    @property
    def p_lo(self):
        return self.p_block()[0]

    @property
    def p_hi(self):
        return self.p_block()[1]

    @property
    def lp(self) -> int:
        return self.p_hi - self.p_lo

    @property
    def q_max(self) -> int:
        return max(b - a for a, b in (self.q_block(t) for t in range(self.world)))

    @property
    def p_max(self) -> int:
        return max(b - a for a, b in (self.p_block(t) for t in range(self.world)))

    def s_max(self, kind: int) -> int:
        return {MOD_DOWN: self.p_max, RESCALE: 2, MERGED: self.p_max + 2}[kind]

    def lq(self, level: int, t: Optional[int] = None) -> int:
        lo, hi = self.q_block(t)
        return max(0, min(hi, level) - lo)

    def q_rows(self, level: int) -> List[int]:
        """global prime indices of the owned Q rows below ``level``"""
        return list(range(self.q_lo, self.q_lo + self.lq(level)))

    def p_rows(self) -> List[int]:
        return [self.L + j for j in range(self.p_lo, self.p_hi)]

    # -- splitting full objects into shard-local ones (host or device tensors) --
    def split_ct(self, ct: torch.Tensor, level: int) -> torch.Tensor:
        """[2][level][n] -> [2][lq][n]"""
        return ct[:, self.q_lo:self.q_lo + self.lq(level)].contiguous()

    def split_poly(self, p: torch.Tensor, level: int) -> torch.Tensor:
        """[level][n] -> [lq][n]"""
        return p[self.q_lo:self.q_lo + self.lq(level)].contiguous()

    def split_key(self, evk: torch.Tensor) -> torch.Tensor:
        """[D][2][L+alpha][n] -> [D][2][(q_hi-q_lo)+(p_hi-p_lo)][n]"""
        q = evk[:, :, self.q_lo:self.q_hi]
        p = evk[:, :, self.L + self.p_lo:self.L + self.p_hi]
        return torch.cat([q, p], dim=2).contiguous()

    def assemble_ct(self, parts: Sequence[torch.Tensor], level: int) -> torch.Tensor:
        """inverse of split_ct over all ranks (parts in rank order)"""
        return torch.cat(list(parts), dim=1)


# --------------------------------------------------------------- exchanges --
class LocalExchange:
    """All shards live in this process (one GPU or CPU): the all-gather is a stack."""

    def all_gather(self, sends: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        g = torch.stack(list(sends))
        return [g] * len(sends)


class TorchExchange:
    """One shard per process; all-gather over ``torch.distributed`` (NCCL over
    NVLink/NVSwitch on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)

    def all_gather(self, sends: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        (send,) = sends
        out = torch.empty((self.world,) + tuple(send.shape), dtype=send.dtype, device=send.device)
        if send.is_cuda:
            self.dist.all_gather_into_tensor(out, send.contiguous(), group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), send.contiguous(), group=self.group)
        return [out]


class LocalPeerExchange:
    """Peer-memory exchange between shards driven from one process (one GPU:
    the 'peers' are the other shards' buffers on the same device)."""
    peer = True

    def __init__(self, backends: Sequence):
        bases = [be.exchange_buffer() for be in backends]
        for be in backends:
            be.set_peers(bases)
        self.backends = list(backends)

    def errors(self) -> List[int]:
        return [be.peer_error() for be in self.backends]

    def close(self):
        pass


class IpcPeerExchange:
    """Peer-memory exchange, one shard per process: every rank exports its
    exchange buffer with CUDA IPC, the handles travel over ``torch.distributed``
    (all_gather_object) and every rank maps its peers' buffers once."""
    peer = True

    def __init__(self, backend, group=None):
        import torch.distributed as dist
        from . import _native as nat
        self.nat, self.backend = nat, backend
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        base = backend.exchange_buffer()
        h = (ctypes.c_ubyte * 64)()
        nat.call("ck_ipc_get_handle", ctypes.c_void_p(base), h)
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h), group=group)
        self.opened = []
        bases = []
        for t, hb in enumerate(handles):
            if t == rank:
                bases.append(base)
                continue
            p = ctypes.c_void_p()
            nat.call("ck_ipc_open_handle", (ctypes.c_ubyte * 64).from_buffer_copy(hb), ctypes.byref(p))
            self.opened.append(p)
            bases.append(p.value)
        backend.set_peers(bases)
        dist.barrier(group=group)

    def errors(self) -> List[int]:
        return [self.backend.peer_error()]

    def close(self):
        for p in self.opened:
            self.nat.call("ck_ipc_close", p)
        self.opened = []


# ---------------------------------------------------------- device backend --
class ShardBackend:
    """One shard on the GPU: the ``ck_shard_*`` C-ABI entry points."""

    def __init__(self, ctx, world: int, rank: int):
        from . import _native as nat
        self.nat, self.ctx = nat, ctx
        h = ctypes.c_void_p()
        nat.call("ck_shard_create", ctx.handle, world, rank, ctypes.byref(h))
        self._h = h
        self.layout = ShardLayout(ctx.params.l, ctx.params.alpha, world, rank)
        lay = (ctypes.c_uint32 * 8)()
        nat.call("ck_shard_layout", h, ctx.params.l, lay)
        got = tuple(lay)
        want = (self.layout.q_lo, self.layout.q_hi, self.layout.p_lo, self.layout.p_hi, self.layout.lq(ctx.params.l),
                self.layout.q_max, self.layout.p_max, world)
        if got != want:
            raise RuntimeError(f"shard layout mismatch: native {got} vs host {want}")

    def close(self):
        if getattr(self, "_h", None):
            self.nat.call("ck_shard_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- peer exchange (send / recv = None in the phase calls) --
    def exchange_buffer(self) -> int:
        base, nbytes = ctypes.c_void_p(), ctypes.c_uint64()
        self.nat.call("ck_shard_exchange_buffer", self._h, ctypes.byref(base), ctypes.byref(nbytes))
        return base.value

    def set_peers(self, bases: Sequence[int]):
        arr = (ctypes.c_uint64 * len(bases))(*bases)
        self.nat.call("ck_shard_set_peers", self._h, arr, len(bases))

    def set_timeout(self, seconds: float):
        self.nat.call("ck_shard_set_timeout", self._h, int(seconds * 1e9))

    def peer_error(self) -> int:
        e = ctypes.c_uint32()
        self.nat.call("ck_shard_peer_error", self._h, ctypes.byref(e))
        return e.value

    def _p(self, t: Optional[torch.Tensor]):
        if t is None:
            return None
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("shard buffers must be contiguous GPU tensors")
        return t.data_ptr()

    def _empty(self, *shape):
        return torch.empty(shape, dtype=torch.int32, device=self.ctx.device)

    def tensor(self, level, x, y):
        lq = self.layout.lq(level)
        d01, d2 = self._empty(2, lq, self.ctx.n), self._empty(lq, self.ctx.n)
        self.nat.call("ck_shard_tensor", self._h, level, self._p(x), self._p(y), self._p(d01), self._p(d2),
                      self.ctx.stream())
        return d01, d2

    def modup_begin(self, level, d, peer=False):
        send = None if peer else torch.zeros((self.layout.q_max, self.ctx.n), dtype=torch.int32,
                                             device=self.ctx.device)
        self.nat.call("ck_shard_modup_begin", self._h, level, self._p(d), self._p(send), self.ctx.stream())
        return send

    def modup_keymult(self, level, recv, d, evk, fold=None):
        rows = self.layout.lq(level) + self.layout.lp
        v = self._empty(2, rows, self.ctx.n)
        self.nat.call("ck_shard_modup_keymult", self._h, level, self._p(recv), self._p(d), self._p(evk),
                      self._p(fold), self._p(v), self.ctx.stream())
        return v

    def switch_begin(self, kind, level, v, peer=False):
        send = None if peer else torch.zeros((2, self.layout.s_max(kind), self.ctx.n), dtype=torch.int32,
                                             device=self.ctx.device)
        self.nat.call("ck_shard_switch_begin", self._h, kind, level, self._p(v), self._p(send), self.ctx.stream())
        return send

    def switch_end(self, kind, level, recv, v, addend=None, add_mask=0, rot=None):
        out_q = level if kind == MOD_DOWN else level - 2
        out = self._empty(2, self.layout.lq(out_q), self.ctx.n)
        self.nat.call("ck_shard_switch_end", self._h, kind, level, self._p(recv), self._p(v), self._p(addend),
                      add_mask, int(rot is not None), int(rot or 0), self._p(out), self.ctx.stream())
        return out


# --------------------------------------------------------------- evaluator --
class LimbShardedEvaluator:
    """Key switching, HMult, HRot and rescale of limb-sharded ciphertexts.

    ``backends`` are the shards this process drives (one per process with
    :class:`TorchExchange`, all of them with :class:`LocalExchange`); every
    per-shard argument is a list in the same order.  Shard-local ciphertexts
    are ``[2][lq][n]`` (see :meth:`ShardLayout.split_ct`), shard-local keys
    ``[D][2][owned Q + owned P][n]`` (:meth:`ShardLayout.split_key`)."""

    def __init__(self, backends: Sequence, exchange, lazy_rescale: bool = False, concurrent: bool = False):
        """``concurrent`` (peer exchange, several shards in this process --
        virtual shards on one GPU): every shard issues its phases on its own
        CUDA stream, so the shards run side by side as they do on separate
        GPUs; the only cross-shard ordering is the exchange's device flags."""
        self.backends = list(backends)
        self.x = exchange
        self.peer = bool(getattr(exchange, "peer", False))
        self.lazy_rescale = lazy_rescale
        self.streams = None
        if concurrent and self.peer and len(self.backends) > 1:
            dev = self.backends[0].ctx.device
            self.streams = [torch.cuda.Stream(dev) for _ in self.backends]

    def _fork(self):
        if self.streams:
            cur = torch.cuda.current_stream(self.backends[0].ctx.device)
            for s in self.streams:
                s.wait_stream(cur)

    def _join(self, outs):
        if self.streams:
            cur = torch.cuda.current_stream(self.backends[0].ctx.device)
            for s in self.streams:
                cur.wait_stream(s)
            for o in outs:  # allocated on a shard stream, consumed on the caller's
                if isinstance(o, torch.Tensor):
                    o.record_stream(cur)
        return outs

    def _each(self, fn, *lists):
        """[fn(backend, *args) for every shard], each on its own stream when concurrent."""
        out = []
        for k, args in enumerate(zip(self.backends, *lists)):
            if self.streams:
                with torch.cuda.stream(self.streams[k]):
                    out.append(fn(*args))
            else:
                out.append(fn(*args))
        return out

    def synchronize(self) -> None:
        """Sync point: wait for the device, then raise if a peer exchange
        timed out.  (A timed-out phase 2 never yields silently wrong rows: the
        shard KeyMult / tail kernels write 0xFFFFFFFF, not a residue, when the
        error word is set -- but only this check turns it into an exception.)"""
        torch.cuda.synchronize(self.backends[0].ctx.device)
        errs = self.x.errors() if hasattr(self.x, "errors") else []
        if any(errs):
            raise RuntimeError(f"limb-sharded peer exchange timed out (error words {errs}); outputs are poisoned")

    def _gather(self, sends):
        if self.peer:  # the rows stay in the peers' exchange buffers
            return [None] * len(sends)
        return self.x.all_gather(sends)

    def key_switch_v(self, level: int, ds, evks, folds=None):
        """ModUp + KeyMult (+ fold): v = [2][lq + lp] per shard (ckks.cpp:680-770)."""
        kw = {"peer": True} if self.peer else {}
        sends = self._each(lambda be, d: be.modup_begin(level, d, **kw), ds)
        recvs = self._gather(sends)
        folds = folds or [None] * len(self.backends)
        return self._each(lambda be, r, d, e, f: be.modup_keymult(level, r, d, e, f), recvs, ds, evks, folds)

    def _switch(self, kind, level, vs, addends=None, add_mask=0, rot=None):
        kw = {"peer": True} if self.peer else {}
        sends = self._each(lambda be, v: be.switch_begin(kind, level, v, **kw), vs)
        recvs = self._gather(sends)
        addends = addends or [None] * len(self.backends)
        return self._each(lambda be, r, v, a: be.switch_end(kind, level, r, v, a, add_mask, rot), recvs, vs, addends)

    def key_switch(self, level: int, ds, evks):
        """key_switch (ckks.cpp:778-787): [2][lq] per shard (c0, c1)."""
        self._fork()
        return self._join(self._switch(MOD_DOWN, level, self.key_switch_v(level, ds, evks)))

    def rescale(self, level: int, cts):
        """rescale (ckks.cpp:789-802): [2][lq(level-2)] per shard."""
        if level < 4:
            raise ValueError("level exhausted")
        self._fork()
        return self._join(self._switch(RESCALE, level, cts))

    def hmult(self, level: int, xs, ys, relins):
        """hmult (ckks.cpp:804-865): merged ModDown + rescale (level - 2), or
        lazy (ModDown, then + (d0, d1), level kept) when ``lazy_rescale``."""
        if level < 4:
            raise ValueError("level exhausted")
        self._fork()
        t = self._each(lambda be, x, y: be.tensor(level, x, y), xs, ys)
        d01 = [a for a, _ in t]
        d2 = [b for _, b in t]
        if not self.lazy_rescale:
            vs = self.key_switch_v(level, d2, relins, folds=d01)
            return self._join(self._switch(MERGED, level, vs))
        vs = self.key_switch_v(level, d2, relins)
        return self._join(self._switch(MOD_DOWN, level, vs, addends=d01, add_mask=3))

    def hrot(self, level: int, cts, r: int, evks):
        """hrot (ckks.cpp:869-897): key-switch a, c0 += b, automorphism on both."""
        self._fork()
        a = self._each(lambda be, ct: ct[1].contiguous(), cts)
        vs = self.key_switch_v(level, a, evks)
        full = self._each(lambda be, ct: ct.contiguous(), cts)
        return self._join(self._switch(MOD_DOWN, level, vs, addends=full, add_mask=1, rot=r))


def exchange_bytes(layout: ShardLayout, n: int, level: int, kind: int) -> int:
    """Bytes one rank receives per mechanism (ModUp + one switch) — the
    all-gather payload of SURVEY §8(e)."""
    up = (layout.world - 1) * layout.q_max * n * 4
    down = (layout.world - 1) * 2 * layout.s_max(kind) * n * 4
    return up + down
