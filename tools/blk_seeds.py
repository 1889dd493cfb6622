"""Blocked sketch (NEXT-3) at full size: lossless rate over hash seeds.

    python tools/blk_seeds.py [config] [seeds] [gamma] [L] [cells_per_block]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import config  # noqa: E402
from paper_2402_07529_b200.sizing import size_blocked  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "vgg"
    seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    gamma = float(sys.argv[3]) if len(sys.argv) > 3 else 1.30
    L = int(sys.argv[4]) if len(sys.argv) > 4 else 256
    cpb = int(sys.argv[5]) if len(sys.argv) > 5 else 12288
    dev = torch.device("cuda", 0)
    wl = config(name, law="gauss")
    xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
    sz, nb = size_blocked(wl.d, wl.density, wl.workers, gamma=gamma, k_bloom=0, L=L, cells_per_block=cpb)
    ok = 0
    rounds = []
    for s in range(seeds):
        p = lhc.params(wl.d, sz.m, sz.c, 3, 0, L, 0x1DC0DE + 104729 * s, nb)
        run = lhc.LosslessAllReduce(p, min(wl.d, int(sz.n_cand_expected * 1.1) + 4096),
                                    local_workers=len(xs), per_worker=False, device=dev)
        dec = run.step(xs)
        torch.cuda.synchronize()
        st = dec.read_stats()
        ok += st["success"]
        rounds.append(st["rounds"])
        print(s, st, flush=True)
    print(f"{name} gamma={gamma} L={L} blocks={nb} c={sz.c}: lossless {ok}/{seeds}, rounds {min(rounds)}-{max(rounds)}")


if __name__ == "__main__":
    main()
