"""Drive the CUDA path (through the C ABI) and the oracle with the same ops and the same generated inputs.

Inputs come only from synth/ (host numpy; the bits are copied to the device for the CUDA side).  No
oracle input and no expected value is ever read back from the CUDA path."""
from __future__ import annotations

import numpy as np
import torch

from oracle import Oracle
from oracle.bf16 import bf16_to_f64
from paper_2510_25412_b200 import kvfs as K
from synth.workloads import TAG_K, TAG_Q, TAG_V, outlier_channels, rows_np

MAX_ABS = 2e-2   # north-star tolerance (BASELINE.json): max-abs error of bf16 attention outputs
MEAN_ABS = 2e-3  # and mean-abs error, fp32 accumulation vs the fp64 oracle


def to_dev(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


def to_host_pinned(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).pin_memory()


def to_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def assert_close(gpu_bf16: np.ndarray, ref: np.ndarray, what=""):
    g = bf16_to_f64(gpu_bf16)
    assert np.isfinite(g).all(), f"{what}: non-finite output"
    err = np.abs(g - ref)
    assert err.max() <= MAX_ABS, f"{what}: max abs err {err.max():.3e}"
    assert err.mean() <= MEAN_ABS, f"{what}: mean abs err {err.mean():.3e}"
    return float(err.max()), float(err.mean())


class Harness:
    def __init__(self, n_pages, P=16, Hq=8, Hkv=2, D=64, L=1, seed=0, max_rows=4096, max_descs=1024,
                 outliers=None):
        """outliers = (channels, k_e, q_e, v_e): channels of every head scaled by 2^k_e in K, 2^q_e in Q and
        2^v_e in V (synth.workloads.outlier_channels; exact, the same bits on both sides)."""
        self.outliers = outliers
        self.c = K.KVFS(L, Hq, Hkv, D, P, n_pages, max_batch_rows=max_rows, max_batch_descs=max_descs, device=0)
        self.o = Oracle(n_pages, P, L, Hkv, D)
        self.L, self.Hq, self.Hkv, self.D, self.P = L, Hq, Hkv, D, P
        self.seed = seed
        self.serial = 0
        self.qserial = 0
        self.fds = {}  # name -> (cfd, ofd)

    def _kv(self, n):
        s0 = self.serial
        self.serial += n
        k = np.stack([rows_np(self.seed, TAG_K, l, 0, s0, s0 + n, self.Hkv * self.D) for l in range(self.L)])
        v = np.stack([rows_np(self.seed, TAG_V, l, 0, s0, s0 + n, self.Hkv * self.D) for l in range(self.L)])
        if self.outliers:
            ch, ke, _, ve = self.outliers
            k, v = outlier_channels(k, self.D, ch, ke), outlier_channels(v, self.D, ch, ve)
        return k.reshape(self.L, n, self.Hkv, self.D), v.reshape(self.L, n, self.Hkv, self.D)

    def _q(self, n, std=1.0):
        s0 = self.qserial
        self.qserial += n
        q = np.stack([rows_np(self.seed, TAG_Q, l, 0, s0, s0 + n, self.Hq * self.D, std) for l in range(self.L)])
        if self.outliers:
            q = outlier_channels(q, self.D, self.outliers[0], self.outliers[2])
        return q.reshape(self.L, n, self.Hq, self.D)

    def open(self, name):
        self.fds[name] = (self.c.open(name), self.o.open(name))

    def append(self, name, pos):
        cfd, ofd = self.fds[name]
        k, v = self._kv(len(pos))
        self.c.append(cfd, pos, to_dev(k), to_dev(v))
        self.o.append(ofd, pos, k, v)

    def fork(self, src, dst):
        self.fds[dst] = (self.c.fork(self.fds[src][0], dst), self.o.fork(self.fds[src][1], dst))

    def truncate(self, name, n):
        self.c.truncate(self.fds[name][0], n)
        self.o.truncate(self.fds[name][1], n)

    def evict(self, name, ranges, compact=False):
        self.c.evict(self.fds[name][0], ranges, compact=compact)
        self.o.evict(self.fds[name][1], ranges, 1 if compact else 0)

    def compact(self, name):
        self.c.compact(self.fds[name][0])
        self.o.compact(self.fds[name][1])

    def unlink(self, name):
        cfd, ofd = self.fds.pop(name)
        self.c.unlink(name)
        self.o.unlink(name)
        self.c.close(cfd)
        self.o.close(ofd)

    def pred(self, rows, qstd=1.0, scale=None, check=True, sentinel=True, host_io=False):
        """rows: list of (name, positions). Runs the batch on both sides; returns (status, out bits, lse).
        host_io: through pred_attn_batch_host with pinned host buffers instead of device tensors."""
        descs_c, descs_o, pos = [], [], []
        for name, ps in rows:
            cfd, ofd = self.fds[name] if name in self.fds else (987, 987)
            descs_c.append((cfd, len(ps)))
            descs_o.append((ofd, len(ps)))
            pos.extend(ps)
        T = len(pos)
        k, v = self._kv(T)
        q = self._q(T, qstd)
        scale = scale if scale is not None else self.D ** -0.5
        assert self.L == 1
        dev = "cpu" if host_io else "cuda"
        out = torch.full((max(T, 1), self.Hq, self.D), float("nan") if sentinel else 0.0, dtype=torch.bfloat16,
                         device=dev)
        lse = torch.full((max(T, 1), self.Hq), float("nan"), dtype=torch.float32, device=dev)
        if host_io:
            out, lse = out.pin_memory(), lse.pin_memory()
            qh, kh, vh = (to_host_pinned(x[0]) if T else None for x in (q, k, v))
            st = self.c.pred_attn_batch_host(descs_c, pos, qh, kh, vh, out if T else None, lse if T else None,
                                             scale=scale)
            self.c.pred_host_fence()
        else:
            st = self.c.pred_attn_batch(descs_c, pos, to_dev(q[0]) if T else None, to_dev(k[0]) if T else None,
                                        to_dev(v[0]) if T else None, out if T else None, lse if T else None,
                                        scale=scale)
        torch.cuda.synchronize()
        st_o, out_o, lse_o = self.o.pred_batch(descs_o, pos, q, k, v, scale)
        assert st == st_o, (st, st_o)
        ob = to_bits(out)[:T]
        lb = lse.cpu().numpy()[:T]
        if check:
            r = 0
            for (name, ps), s in zip(rows, st):
                n = len(ps)
                if s == 0 and n:
                    assert_close(ob[r:r + n], out_o[0, r:r + n], f"pred {name}")
                    np.testing.assert_allclose(lb[r:r + n], lse_o[0, r:r + n], atol=2e-3, rtol=0)
                elif n:
                    assert np.isnan(bf16_to_f64(ob[r:r + n])).all(), "failed descriptor rows must be untouched"
                r += n
        return st, ob, lb, out_o[0], lse_o[0]

    def check_meta(self):
        assert self.c.refcounts() == self.o.refcnt
        for name, (cfd, ofd) in self.fds.items():
            assert self.c.table(cfd) == self.o.table(ofd), name
            assert self.c.positions(cfd) == self.o.positions(ofd), name
        self.c.audit()

    def check_data(self):
        """kvfs_read of every file equals the oracle's retained K/V bits (bit-exact)."""
        for name, (cfd, ofd) in self.fds.items():
            n = self.o.stat(ofd)[0]
            for layer in range(self.L):
                if n == 0:
                    continue
                kk, vv = self.c.read(cfd, layer, 0, n)
                ko, vo = self.o.read(ofd, layer, 0, n)
                assert np.array_equal(to_bits(kk), ko), name
                assert np.array_equal(to_bits(vv), vo), name


def scores_rtol(q_f64: np.ndarray, k_f64: np.ndarray, lse_gpu: np.ndarray, lse_ref: np.ndarray, scale: float):
    """Per-key relative error bound of the K9 scores of one descriptor.

    score_k = sum_{i,h} w_{k,i,h}, w = exp(s - lse), every term positive.  The kernel takes the SAME bf16 Q/K
    bits as the oracle and the lse that the attention kernel wrote, so each w carries at most
      |d lse_{i,h}|                    (the attention kernel's lse error: measured here, <= 2e-3 by the lse check)
    + gamma_D * scale * |q_{i,h}| |k|  (fp32 accumulation of the D-term dot product, Cauchy-Schwarz bound;
                                        gamma_D = D * 2^-24)
    + 2^-21                            (MUFU ex2.approx relative error, incl. the fp32 log2(e) folding)
    of relative error in the exponent, and the fp32 sum of n_q * Hq positive terms adds n_q * Hq * 2^-24
    relative.  So |got_k - ref_k| <= rtol * ref_k with the rtol returned here (first order; expm1 keeps it
    an upper bound).  q_f64 [n_q][Hq][D], k_f64 [len][Hkv][D]; lse_* [n_q][Hq]."""
    n_q, hq, d = q_f64.shape
    dlse = float(np.abs(np.asarray(lse_gpu, np.float64) - np.asarray(lse_ref, np.float64)).max())
    qn = float(np.sqrt((q_f64 ** 2).sum(-1)).max())
    kn = float(np.sqrt((k_f64 ** 2).sum(-1)).max())
    ds = d * 2.0 ** -24 * scale * qn * kn
    return float(np.expm1(dlse + ds + 2.0 ** -21) + n_q * hq * 2.0 ** -24)
