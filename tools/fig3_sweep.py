"""The paper's recovery experiment (§4.1.1, Fig. `exp::recovery`) as a
measurement of the GPU path, plus the §8(d) VGG19 provisioning sweep.

(1) Fig. 3 analogue: one worker, VGG19-sized gradient (d = 143 M) at Table 1's
    sparsity (30.4 %: 69.6 % nonzero), exact bitmap index, counter
    cells c swept as a fraction of d ("compressed data size", reading R16) from 2 %
    to 200 %; 20 hash seeds per point.  Per point: the paper's three metrics —
    average relative error (mean over the nonzero parameters of |x^ - x| / |x|),
    recovery rate (fraction of candidates recovered by peeling) and recovery
    iterations (synchronous rounds) — as mean and range over the seeds.  The paper's
    threshold is gamma (1 - sparsity) = 1.23 x 0.696 = 85.6 %.
(2) The §8(d) sweep at the BASELINE VGG19 config (d = 143 M, 1 %, 8 workers, Bloom
    index): gamma_s = 1.10 ... 1.50, 20 hash seeds each: success rate and rounds.
(3) Oracle spot checks: the same experiment scaled to d = 2 M at three c/d points,
    two seeds each, GPU against the CPU oracle (flags and rounds bit-exact, values
    within the north-star tolerance).

    python tools/fig3_sweep.py [--seeds 20] [--out profiles/r02_fig3.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from lhc_inputs import config, rng_for, values  # noqa: E402
from paper_2402_07529_b200.sizing import INDEX_BITMAP  # noqa: E402

FRACS = [0.02, 0.1, 0.3, 0.5, 0.6, 0.7, 0.75, 0.8, 0.83, 0.85, 0.856, 0.87, 0.9, 0.95,
         1.0, 1.1, 1.2, 1.5, 2.0]
GAMMAS = [1.10, 1.15, 1.20, 1.22, 1.25, 1.30, 1.40, 1.50]


def table1_input(d, density, seed, dev):
    rng = rng_for(seed)
    nnz = int(round(density * d))
    idx = np.sort(rng.choice(d, nnz, replace=False)).astype(np.int64)
    x = np.zeros(d, np.float32)
    x[idx] = values(rng, nnz, "gauss", 1e-3)
    return torch.from_numpy(x).to(dev)


def decode_point(p, x, dev, cap):
    run = lhc.LosslessAllReduce(p, cap_cand=cap, local_workers=1, device=dev)
    dec = run.step([x])
    torch.cuda.synchronize()
    st = dec.read_stats()
    nz = x != 0
    rel = ((dec.dense[nz] - x[nz]).abs() / x[nz].abs()).mean().item()
    return st, rel


def fig3(seeds, dev, d=143_000_000, density=0.696):
    L = 1024
    m = -(-d // L) * L
    x = table1_input(d, density, 3040, dev)
    out = []
    for frac in FRACS:
        c = max(3 * L, int(round(frac * d / (3 * L))) * 3 * L)
        rows = []
        for s in range(seeds):
            p = lhc.params(d, m, c, 3, INDEX_BITMAP, L, 0xF16 + 7919 * s)
            st, rel = decode_point(p, x, dev, d)
            rows.append((st["n_peeled"] / max(1, st["n_cand"]), rel, st["rounds"], st["success"]))
        rate, rel, rnd, succ = (np.array(v, dtype=np.float64) for v in zip(*rows))
        pt = {"c_over_d": c / d, "rate_mean": rate.mean(), "rate_min": rate.min(), "rate_max": rate.max(),
              "rel_err_mean": rel.mean(), "rel_err_max": rel.max(), "rounds_mean": rnd.mean(),
              "rounds_min": int(rnd.min()), "rounds_max": int(rnd.max()), "success_frac": succ.mean()}
        print(json.dumps(pt), flush=True)
        out.append(pt)
    return {"d": d, "density": density, "workers": 1, "index": "bitmap", "k": 3, "L": L,
            "seeds": seeds, "threshold_paper": 1.23 * (1 - 0.304), "points": out}


def gamma_sweep(seeds, dev):
    wl = config("vgg", law="gauss")
    xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
    out = []
    for g in GAMMAS:
        s = lhc.size_workload(wl.d, wl.density, wl.workers, gamma=g)
        rows = []
        for k in range(seeds):
            p = lhc.params(wl.d, s.m, s.c, 3, 0, 1024, 0x1DC0DE + 104729 * k)
            run = lhc.LosslessAllReduce(p, min(wl.d, int(s.n_cand_expected * 1.1) + 4096),
                                        local_workers=wl.workers, per_worker=False, device=dev)
            dec = run.step(xs)
            torch.cuda.synchronize()
            st = dec.read_stats()
            rows.append((st["success"], st["rounds"], st["n_peeled"] / max(1, st["n_cand"])))
        succ, rnd, rate = (np.array(v, dtype=np.float64) for v in zip(*rows))
        pt = {"gamma_s": g, "c": int(s.c), "success_frac": succ.mean(), "rounds_mean": rnd.mean(),
              "rounds_min": int(rnd.min()), "rounds_max": int(rnd.max()), "rate_min": rate.min()}
        print(json.dumps(pt), flush=True)
        out.append(pt)
    return {"config": "vgg (d=143M, 1%, 8 workers, Bloom k_B=3, L=1024)", "seeds": seeds, "points": out}


def spot_checks(dev):
    import oracle

    oracle.build()
    d, density, L = 2_000_000, 0.696, 1024
    m = -(-d // L) * L
    x = table1_input(d, density, 77, dev)
    xh = x.cpu().numpy()
    res = []
    for frac in (0.7, 0.856, 1.0):
        c = int(round(frac * d / (3 * L))) * 3 * L
        for s in range(2):
            p = lhc.params(d, m, c, 3, INDEX_BITMAP, L, 0x5B07 + s)
            run = lhc.LosslessAllReduce(p, cap_cand=d, local_workers=1, device=dev)
            dec = run.step([x])
            torch.cuda.synchronize()
            st = dec.read_stats()
            op = oracle.params(d, m, c, 3, INDEX_BITMAP, L, p.seed)
            _, _, ref = oracle.pipeline(op, [xh])
            n = st["n_cand"]
            val = dec.val[:n].cpu().numpy().astype(np.float64)
            ok = (n == ref.stats.n_cand and st["rounds"] == ref.stats.rounds
                  and st["success"] == ref.stats.success
                  and np.array_equal(dec.peeled[:n].cpu().numpy().astype(bool), ref.peeled)
                  and bool(np.all(np.abs(val - ref.val) <= 1e-7 + 1e-5 * np.abs(ref.val))))
            res.append({"c_over_d": c / d, "seed": s, "rounds": st["rounds"],
                        "rate": st["n_peeled"] / max(1, n), "match": bool(ok)})
            print(json.dumps(res[-1]), flush=True)
    return {"d": d, "density": density, "checks": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_fig3.json"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    t0 = time.time()
    doc = {"what": "recovery metrics vs compressed size (P:L322-344) and the VGG19 gamma sweep, "
                   "measured on the GPU path; oracle spot checks at d = 2 M",
           "fig3": fig3(args.seeds, dev), "gamma_sweep": gamma_sweep(args.seeds, dev),
           "oracle_spot_checks": spot_checks(dev)}
    doc["wall_s"] = time.time() - t0
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
