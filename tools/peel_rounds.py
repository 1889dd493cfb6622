"""Per-round times of the frontier peel (k_peel built with -DLHC_PEEL_TIMING=1, loaded
through LHC_LIB): round r's frontier size (Ctrl.fsize) and its duration (Ctrl.t).

    LHC_LIB=scratch/liblhc_ptime.so python tools/peel_rounds.py [config ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import config  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:] or ["vgg"]:
        wl = config(name, law="gauss")
        s = lhc.size_workload(wl.d, wl.density, wl.workers)
        p = lhc.params(wl.d, s.m, s.c, 3, 0, 1024, 0x1DC0DE)
        xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
        run = lhc.LosslessAllReduce(p, min(wl.d, int(s.n_cand_expected * 1.05) + 4096),
                                    local_workers=len(xs), per_worker=False, device=dev)
        for _ in range(3):
            run.step(xs)
        torch.cuda.synchronize()
        raw = run.decoder.ws[:16384].cpu().numpy().tobytes()
        off_t = 96
        t = np.frombuffer(raw[off_t:off_t + 128 * 8], dtype=np.uint64).astype(np.int64)
        fs = np.frombuffer(raw[off_t + 1024:off_t + 1024 + 512], dtype=np.uint32)
        print(f"== {name}: init {(t[2]-t[0])/1e3:.1f} us, F0 {(t[3]-t[2])/1e3:.1f} us, "
              f"rounds to end {(t[127]-t[3])/1e3:.1f} us, "
              f"finalize {((t[1]-t[127])/1e3 if t[1] else float('nan')):.1f} us, stats {run.decoder.read_stats()}")
        rows = []
        for r in range(1, 100):
            if not t[r + 3]:
                break
            nxt = t[r + 4] if t[r + 4] else (t[126] if t[126] else t[127])
            rows.append(f"{r}:{fs[r]}/{(nxt - t[r + 3]) / 1e3:.1f}us")
        print("   round:entries/time", " ".join(rows))
        if t[126]:  # two-pass peel: t[126] = end of pass 1, t[127] = end of pass 2
            print(f"   pass 1 {(t[126] - t[3]) / 1e3:.1f} us, pass 2 {(t[127] - t[126]) / 1e3:.1f} us")
            o2 = off_t + 128 * 8 + 512 + 1024  # Ctrl.tflush: pass-2 segment starts
            tf = np.frombuffer(raw[o2:o2 + 1024], dtype=np.uint64).astype(np.int64)
            n = int(np.count_nonzero(tf))
            seg = [(tf[s + 1] if s + 1 < n else t[127]) - tf[s] for s in range(n)]
            print("   pass 2 segment times (us):", " ".join(f"{x / 1e3:.1f}" for x in seg))


if __name__ == "__main__":
    main()
