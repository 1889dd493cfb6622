"""Peel diagnostics on one GPU: per-launch times of the decode (CUDA events between
the launches of sketch_query / sketch_peel) and the peel kernel's own device
timestamps (Ctrl.t: init, start of every round, end of the rounds).

    python tools/peel_diag.py [config ...]        (e.g. ncf vgg)
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import config  # noqa: E402


def main():
    names = sys.argv[1:] or ["ncf"]
    dev = torch.device("cuda", 0)
    for name in names:
        wl = config(name, law="gauss")
        s = lhc.size_workload(wl.d, wl.density, wl.workers)
        p = lhc.params(wl.d, s.m, s.c, 3, 0, 1024, 0x1DC0DE)
        xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
        run = lhc.LosslessAllReduce(p, min(wl.d, int(s.n_cand_expected * 1.05) + 4096),
                                    local_workers=len(xs), device=dev)
        for _ in range(3):
            run.step(xs)
        torch.cuda.synchronize()
        dec = run.decoder
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        dec.query(run.sketch)
        ev[1].record()
        dec.peel(run.sketch)
        ev[2].record()
        torch.cuda.synchronize()
        st = dec.read_stats()
        # Ctrl sits at offset 0 of the workspace: n_cand u64, overflow u32, rc[3] u64 (8-aligned),
        # rounds_dbg, compact_fail, blk_fail, blk_done u32, blk_peeled u64, blk_rounds u32,
        # xl_n[2], yl_n[2] u32, t[128] u64
        raw = dec.ws[:16384].cpu().numpy().tobytes()
        off_t = 96
        t = np.frombuffer(raw[off_t:off_t + 128 * 8], dtype=np.uint64).astype(np.int64)
        print(f"== {name}: query {ev[0].elapsed_time(ev[1])*1e3:.1f} us, peel (all launches) "
              f"{ev[1].elapsed_time(ev[2])*1e3:.1f} us; stats {st}")
        t0 = t[0]
        if t0:
            marks = [("init", t[2])] + [(f"r{r}", t[r + 3]) for r in range(1, 120) if t[r + 3]] + \
                    [("end", t[127])]
            prev = t0
            line = []
            for nm, v in marks:
                if v:
                    line.append(f"{nm}:{(v - prev) / 1e3:.1f}")
                    prev = v
            print("   kernel phases (us since previous mark):", " ".join(line))
            print(f"   kernel total to end of rounds: {(t[127] - t0) / 1e3:.1f} us")
            # Ctrl: ... t[128] u64, fsize[128] u32, tproc[128] u64, tflush[128] u64
            o2 = off_t + 128 * 8
            fs = np.frombuffer(raw[o2:o2 + 128 * 4], dtype=np.uint32)
            tp = np.frombuffer(raw[o2 + 512:o2 + 512 + 1024], dtype=np.uint64).astype(np.int64)
            tf = np.frombuffer(raw[o2 + 1536:o2 + 1536 + 1024], dtype=np.uint64).astype(np.int64)
            o3 = o2 + 1536 + 1024
            dbg = np.frombuffer(raw[o3:o3 + 4 * 1024], dtype=np.uint64).reshape(4, 128).astype(np.int64)
            for r in range(1, 40):
                if not t[r + 3]:
                    break
                print(f"   round {r}: X sum {dbg[1][r] / 1965:.0f} us-warp, Y sum {dbg[3][r] / 1965:.0f} us-warp")
                print(f"   round {r}: X last warp {(tp[r] - t[r + 3]) / 1e3:8.1f} us, X barrier exit "
                      f"{fs[r] / 10:8.1f} us, Y last warp {(tf[r] - t[r + 3]) / 1e3:8.1f} us")
        # per-launch breakdown with LHC_PEEL_TIMING-free events: time each launch class
        for impl in ("frontier", "frontier"):
            os.environ["LHC_PEEL_IMPL"] = impl
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dec.query(run.sketch)
            e0.record()
            dec.peel(run.sketch)
            e1.record()
            torch.cuda.synchronize()
            print(f"   LHC_PEEL_IMPL={impl}: peel {e0.elapsed_time(e1)*1e3:.1f} us {dec.read_stats()}")
        os.environ.pop("LHC_PEEL_IMPL")


if __name__ == "__main__":
    main()
