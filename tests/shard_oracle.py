"""TEST INFRASTRUCTURE ONLY: a limb-shard backend computed with the C oracle
(oracle/pyoracle.py) on CPU tensors, with the same phase semantics as the
native ``ck_shard_*`` entry points.  It lets the CPU tests drive
``paper_2407_13055_b200.limb.LimbShardedEvaluator`` — partition, send/recv
layouts and the all-gather over gloo — without a GPU, and check the result
against the oracle's single-host mechanisms.  Never used by the product."""
from __future__ import annotations

import numpy as np
import torch

from paper_2407_13055_b200.limb import MERGED, MOD_DOWN, RESCALE, ShardLayout

R32 = 1 << 32


class OracleShard:
    def __init__(self, oracle, world: int, rank: int):
        self.O = oracle
        self.layout = ShardLayout(oracle.l, oracle.alpha, world, rank)
        self.q = oracle.primes.astype(np.int64)

    # -- helpers --
    def _qcol(self, gs):
        return self.q[np.asarray(gs, np.int64)][:, None]

    def _rinv(self, gs):
        return np.array([pow(R32 % int(self.q[g]), -1, int(self.q[g])) for g in gs], np.int64)[:, None]

    def _mont(self, a, b, gs):  # a*b*R^-1 mod q, canonical inputs
        q = self._qcol(gs)
        return (a.astype(np.int64) * b.astype(np.int64) % q) * self._rinv(gs) % q

    def _canon(self, a, gs):
        return self.O.canonical(np.asarray(a), np.asarray(gs, np.uint32)).astype(np.int64)

    def _sources(self, kind, level):
        L, A = self.O.l, self.O.alpha
        if kind == MOD_DOWN:
            return [L + j for j in range(A)], level
        sg = [level - 2, level - 1] + ([L + j for j in range(A)] if kind == MERGED else [])
        return sg, level - 2

    def _owns(self, t, g):
        if g < self.O.l:
            lo, hi = self.layout.q_block(t)
            return lo <= g < hi
        lo, hi = self.layout.p_block(t)
        return lo <= g - self.O.l < hi

    def _local_row(self, level, g):
        lay = self.layout
        return g - lay.q_lo if g < self.O.l else lay.lq(level) + (g - self.O.l - lay.p_lo)

    @staticmethod
    def _t(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.int64).astype(np.int32))

    # -- phases (see include/ck32_b200.h, ck_shard_*) --
    def tensor(self, level, x, y):
        gs = self.layout.q_rows(level)
        xb, xa, yb, ya = x[0].numpy(), x[1].numpy(), y[0].numpy(), y[1].numpy()
        q = self._qcol(gs)
        d0 = self._mont(xb, yb, gs)
        d1 = (self._mont(xb, ya, gs) + self._mont(xa, yb, gs)) % q
        d2 = self._mont(xa, ya, gs)
        return self._t(np.stack([d0, d1])), self._t(d2)

    def modup_begin(self, level, d):
        lay, A = self.layout, self.O.alpha
        send = np.zeros((lay.q_max, self.O.n), np.int64)
        for r, g in enumerate(lay.q_rows(level)):
            k = g // A
            sg = list(range(k * A, min((k + 1) * A, level)))
            p1 = self.O.bconv_part1(sg)[g - k * A]
            send[r] = self._canon(self.O.intt(d[r].numpy()[None], [g], [p1]), [g])[0]
        return self._t(send)

    def modup_keymult(self, level, recv, d, evk, fold=None):
        lay, A, n = self.layout, self.O.alpha, self.O.n
        recv = recv.numpy()
        compact = np.zeros((level, n), np.int64)
        for t in range(lay.world):
            lo, _ = lay.q_block(t)
            cnt = lay.lq(level, t)
            compact[lo:lo + cnt] = recv[t, :cnt]
        gl = lay.q_rows(level) + lay.p_rows()
        lq = lay.lq(level)
        D = self.O.digits(level)
        d = d.numpy()
        evk = evk.numpy()
        q = self._qcol(gl)
        v = np.zeros((2, len(gl), n), np.int64)
        erow = [r if r < lq else (lay.q_hi - lay.q_lo) + (r - lq) for r in range(len(gl))]
        for k in range(D):
            b, e = k * A, min((k + 1) * A, level)
            sg = list(range(b, e))
            others = [(r, g) for r, g in enumerate(gl) if not (b <= g < e)]
            opnd = np.zeros((len(gl), n), np.int64)
            if others:
                dg = [g for _, g in others]
                conv = self._canon(self.O.bconv(compact[b:e].astype(np.int32), sg, dg), dg)
                conv = self._canon(self.O.ntt_fwd(conv.astype(np.int32), dg), dg)
                for i, (r, _) in enumerate(others):
                    opnd[r] = conv[i]
            for r, g in enumerate(gl):
                if b <= g < e:
                    opnd[r] = d[r]
            for c in range(2):
                key = evk[k, c][erow]
                v[c] = (v[c] + self._mont(opnd, key, gl)) % q
        if fold is not None and lq:
            f = fold.numpy().astype(np.int64)
            qq = self._qcol(gl[:lq])
            pm = np.array([int(np.prod([int(self.q[self.O.l + j]) % int(self.q[g]) for j in range(A)], dtype=object))
                           % int(self.q[g]) for g in gl[:lq]], np.int64)[:, None]
            for c in range(2):
                v[c, :lq] = (v[c, :lq] + f[c] * pm % qq) % qq
        return self._t(v)

    def switch_begin(self, kind, level, v):
        sg, _ = self._sources(kind, level)
        own = [g for g in sg if self._owns(self.layout.rank, g)]
        p1 = dict(zip(sg, self.O.bconv_part1(sg)))
        send = np.zeros((2, self.layout.s_max(kind), self.O.n), np.int64)
        v = v.numpy()
        for c in range(2):
            for u, g in enumerate(own):
                row = v[c, self._local_row(level, g)]
                send[c, u] = self._canon(self.O.intt(row[None], [g], [p1[g]]), [g])[0]
        return self._t(send)

    def switch_end(self, kind, level, recv, v, addend=None, add_mask=0, rot=None):
        lay, n = self.layout, self.O.n
        sg, out_q = self._sources(kind, level)
        recv = recv.numpy()
        gathered, blocks = [], [[], []]
        for t in range(lay.world):
            own_t = [g for g in sg if self._owns(t, g)]
            gathered += own_t
            for c in range(2):
                blocks[c].append(recv[t, c, :len(own_t)])
        dg = lay.q_rows(out_q)
        if not dg:
            return torch.zeros((2, 0, n), dtype=torch.int32)
        q = self._qcol(dg)
        dinv = np.array([pow(int(np.prod([int(self.q[g]) % int(self.q[i]) for g in sg], dtype=object)) % int(self.q[i]),
                             -1, int(self.q[i])) for i in dg], np.int64)[:, None]
        v = v.numpy().astype(np.int64)
        out = np.zeros((2, len(dg), n), np.int64)
        for c in range(2):
            src = np.concatenate(blocks[c]).astype(np.int32)
            conv = self._canon(self.O.bconv(src, gathered, dg), dg)
            conv = self._canon(self.O.ntt_fwd(conv.astype(np.int32), dg), dg)
            out[c] = (v[c, :len(dg)] - conv + q) % q * dinv % q
            if addend is not None and (add_mask >> c) & 1:
                out[c] = (out[c] + addend[c].numpy().astype(np.int64)) % q
        if rot is not None:
            out = out[:, :, self.O.rotation_src_map(rot).astype(np.int64)]
        return self._t(out)
