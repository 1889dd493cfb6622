"""Blocked-sketch decode diagnostics (NEXT-3): per-block phase times of
k_peel_blocked (build with -DLHC_BLK_TIMING=1, loaded through LHC_LIB).

    LHC_LIB=scratch/liblhc_blkt.so python tools/blk_diag.py [vgg bert ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import config  # noqa: E402
from paper_2402_07529_b200.sizing import size_blocked  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:] or ["vgg"]:
        wl = config(name, law="gauss")
        L = int(os.environ.get("BLK_L", "256"))
        cpb = int(os.environ.get("BLK_CELLS", "12288"))
        sz, nb = size_blocked(wl.d, wl.density, wl.workers, gamma=1.30, k_bloom=0, L=L,
                              cells_per_block=cpb)
        p = lhc.params(wl.d, sz.m, sz.c, 3, 0, L, 0x1DC0DE, nb)
        xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
        run = lhc.LosslessAllReduce(p, min(wl.d, int(sz.n_cand_expected * 1.05) + 4096),
                                    local_workers=len(xs), per_worker=False, device=dev)
        for _ in range(3):
            run.step(xs)
        torch.cuda.synchronize()
        dec = run.decoder
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        dec.query(run.sketch)
        e[1].record()
        dec.peel(run.sketch)
        e[2].record()
        torch.cuda.synchronize()
        raw = dec.ws[:16384].cpu().numpy().tobytes()
        t = np.frombuffer(raw[96:96 + 128 * 8], dtype=np.uint64).astype(np.int64)
        nblk = max(1, t[12])
        print(f"== {name}: blocks={nb} c={sz.c} query {e[0].elapsed_time(e[1])*1e3:.1f} us, peel "
              f"{e[1].elapsed_time(e[2])*1e3:.1f} us, stats {dec.read_stats()}")
        print(f"   per block (mean over {nblk}): load {t[8]/nblk/1e3:.1f} us, insert {t[9]/nblk/1e3:.1f}, "
              f"rounds {t[10]/nblk/1e3:.1f}, finalize+out {t[11]/nblk/1e3:.1f}")
        # Ctrl: t[128] u64 at 96, fsize[128] u32, tproc[128] u64, tflush[128] u64
        o2 = 96 + 128 * 8 + 128 * 4
        tp = np.frombuffer(raw[o2:o2 + 1024], dtype=np.uint64).astype(np.int64)
        tf = np.frombuffer(raw[o2 + 1024:o2 + 2048], dtype=np.uint64).astype(np.int64)
        print("   per round (us per block, peeled per block):",
              " ".join(f"{r}:{tp[r]/nblk/1e3:.2f}/{tf[r]/nblk:.0f}" for r in range(1, 40) if tp[r]))


if __name__ == "__main__":
    main()
