"""Small cases that launch every kernel of libkvfs.so, for compute-sanitizer (memcheck / racecheck / synccheck
/ initcheck, SPEC.md S:144 concurrency model):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Covers: K1 decode (D 64 and 128, fused append, split merge), K2 chunk attention (tcgen05) and K2 prefix mode
(cascade), K9 scores, K4 copy-on-write / fork tail copies (prologue), K5 compaction (single file and the
kvfs_compact_files PDL chain), K6 pack / unpack and the host tier, K7 read, K8 extract / merge gather, the
kvfs_append scatter.  Every result is checked against the oracle, so a run that the sanitizer passes is
also a correct run.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    import __graft_entry__ as ge
    from gpu_harness import Harness, assert_close, to_bits, to_dev  # noqa: F401
    from paper_2510_25412_b200 import kvfs as K

    ge.smoke()  # K1 (D 64), cascade (K2 prefix + K1 merge), K2 chunk, K9 scores
    for (P, Hq, Hkv, D) in ((16, 8, 2, 64), (16, 32, 8, 128)):
        h = Harness(1200, P, Hq, Hkv, D, seed=5)
        h.c.set_option(K.OPT_CASCADE_MIN_ENTRIES, 2)
        h.open("a")
        h.append("a", list(range(300)))
        h.fork("a", "b")                     # full tail: shared pages
        h.open("c")
        h.append("c", list(range(70)))
        h.fork("c", "d")                     # tail with room: K4 tail copy
        h.pred([("b", [300]), ("d", [70, 71, 72]), ("c", [70])])   # CoW on d's shared tail? (fork copied it)
        h.truncate("a", 250)
        h.pred([("a", [250])])               # CoW of the shared tail page after truncate
        h.evict("a", [(3, 40), (100, 131)])
        h.evict("b", [(0, 5)], compact=True)  # K5 single file
        for nm in ("e", "f", "g"):
            h.open(nm)
            h.append(nm, list(range(200)))
            h.evict(nm, [(10, 90)])
        done = h.c.compact_files([h.fds[n][0] for n in ("e", "f", "g")])  # K5 PDL chain
        assert done == 3
        for n in ("e", "f", "g"):
            h.o.compact(h.fds[n][1])
        rows = [("a", [251]), ("b", [301])]
        if D == 128:
            rows.append(("c", list(range(71, 71 + 20))))  # K2 chunk rows
        h.pred(rows)
        h.check_meta()
        h.check_data()                       # K7 read of every file
        # K8 extract / merge
        ex_c = h.c.extract(h.fds["c"][0], [0, 5, 6, 7, 40], "x")
        ex_o = h.o.extract(h.fds["c"][1], [0, 5, 6, 7, 40], "x")
        h.fds["x"] = (ex_c, ex_o)
        h.open("m1")
        h.append("m1", [1000, 1002])
        mc = h.c.merge([h.fds["m1"][0], h.fds["x"][0]], "mm")
        mo = h.o.merge([h.fds["m1"][1], h.fds["x"][1]], "mm")
        h.fds["mm"] = (mc, mo)
        # K6: host tier round trip and pack / unpack into a second ctx
        h.c.offload(h.fds["g"][0])
        h.o.offload(h.fds["g"][1])
        h.c.restore(h.fds["g"][0])
        h.o.restore(h.fds["g"][1])
        torch.cuda.synchronize()
        h.check_meta()
        h.check_data()
        hdr, buf = h.c.pack([h.fds[n][0] for n in ("a", "b")])
        dst = K.KVFS(1, Hq, Hkv, D, P, 600, device=0)
        fds = dst.unpack(hdr, buf, ["a", "b"])
        torch.cuda.synchronize()
        for n, fd in zip(("a", "b"), fds):
            ln = h.o.stat(h.fds[n][1])[0]
            k, v = dst.read(fd, 0, 0, ln)
            ko, vo = h.o.read(h.fds[n][1], 0, 0, ln)
            assert np.array_equal(to_bits(k), ko) and np.array_equal(to_bits(v), vo)
        # K9 scores after the cascade / chunk step
        last = h.o.stat(h.fds["a"][1])[2]
        step, st = h.c.pred_step_begin([(h.fds["a"][0], 1)], [last + 1])
        q = torch.randn((1, Hq, D), device="cuda").to(torch.bfloat16)
        kn = torch.randn((1, Hkv, D), device="cuda").to(torch.bfloat16)
        out = torch.empty((1, Hq, D), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((1, Hq), dtype=torch.float32, device="cuda")
        h.c.pred_attn_layer(step, 0, q, kn, kn, out, lse)
        sc = torch.empty(h.o.stat(h.fds["a"][1])[0] + 1, dtype=torch.float32, device="cuda")
        h.c.pred_attn_scores(step, 0, q, lse, sc, np.zeros(1, np.int64))
        h.c.pred_step_end(step)
        torch.cuda.synchronize()
        assert abs(float(sc.sum()) - Hq) < 1e-2
        if D == 128:
            # cascade variants of round 2: folded split records (S = 2) and the paired partition (a CTA running
            # two prefix units in turn), then the host-buffer pred
            h.open("r")
            h.append("r", list(range(700)))
            for kid in ("r1", "r2", "r3"):
                h.fork("r", kid)
            for splits, paired in ((2, 0), (0, 2)):
                h.c.set_option(K.OPT_PREFIX_SPLITS, splits)
                h.c.set_option(K.OPT_PREFIX_PAIRED, paired)
                rows = []
                for nm in ("r", "r1", "r2", "r3"):
                    rows.append((nm, [h.o.stat(h.fds[nm][1])[2] + 1]))
                h.pred(rows)
            h.c.set_option(K.OPT_PREFIX_SPLITS, 0)
            h.c.set_option(K.OPT_PREFIX_PAIRED, 0)
            h.pred([(nm, [h.o.stat(h.fds[nm][1])[2] + 1]) for nm in ("r", "r2", "c")], host_io=True)
            # (no check_meta here: the K9 step above appended to "a" on the CUDA side only)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
