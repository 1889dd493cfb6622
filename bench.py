#!/usr/bin/env python
"""Benchmark of the lossless homomorphic compression hot path on B200.

One step = Alg. 1 end to end for the configured workload: every
rank compresses the gradients of the workers it holds (W workers spread over N
GPUs), the sketches are aggregated (on one GPU with sketch_aggregate, across
GPUs with the NVLink P2P sketch_allreduce), and every rank decodes the aggregate
into the dense sum.  Metric (BASELINE.json): aggregated gradient elements/s =
d / T_step, d counted once however many workers (footnote P:L367).

    python bench.py [--gpus N --steps K --warmup W --config vgg]
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...     # the CPU oracle, timed as it stands

Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from lhc_inputs import config as workload_config  # noqa: E402

METRIC = "aggregated gradient elements/s (compress+aggregate+decode) at 1/2/4/8 B200"
UNIT = "elements/s"
SEED = 0x1DC0DE


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="vgg",
                    help="tiny|ncf|lstm|bert|vgg (default: VGG19-shaped, the largest single-GPU "
                         "config: d = 143 M, 1 %%, W = 8)")
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--gamma", type=float, default=1.30)
    ap.add_argument("--law", default="gauss")
    ap.add_argument("--index", choices=["bloom", "bitmap", "auto"], default="bloom",
                    help="Bloom filter (default), exact bitmap (P:L188), or the smaller of the two")
    ap.add_argument("--blocks", default="0",
                    help="0: one Count Sketch (default); N or 'auto': the sketch split into "
                         "blocks (P:L206, NEXT-3) peeled block-locally in shared memory")
    ap.add_argument("--L", type=int, default=1024, help="batch width (paper: 1024, P:L261)")
    ap.add_argument("--block-cells", type=int, default=12288, help="cells per block for --blocks auto")
    ap.add_argument("--per-worker", action="store_true",
                    help="one sketch per local worker, cleared and aggregated on the GPU (the "
                         "default compresses a rank's workers straight into its sketch: Y and B "
                         "are homomorphic, P:L137, so the local aggregation is the reductions)")
    ap.add_argument("--fuse-local", action="store_true", help="(the default; kept for old command lines)")
    ap.add_argument("--comm", choices=["p2p", "nvls", "nccl"], default="p2p",
                    help="p2p: NVLink peer stores (two-shot); nvls: NVSwitch multicast "
                         "(in-switch reduction, NEXT-2); nccl: the NCCL baseline")
    ap.add_argument("--decode", choices=["auto", "replicated", "sharded"], default="auto",
                    help="replicated: all-reduce, every rank decodes all of d; sharded: "
                         "per-shard sub-sketches, reduce-scatter, every rank decodes its shard, "
                         "all-gather of the decoded lists (NEXT-2; the paper's 'distributed load "
                         "of the recovery process', P:L380); auto (default): replicated on one "
                         "GPU, sharded on several.  Every rank ends with the same dense sum.")
    ap.add_argument("--deterministic", action="store_true",
                    help="decode with sketch_peel_det (values bit-identical across runs and ranks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel from the host")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--phases", action="store_true", help="also print per-phase times (stderr)")
    return ap.parse_args()


def workload(args):
    over = {"law": args.law}
    if args.density is not None:
        over["density"] = args.density
    if args.workers is not None:
        over["workers"] = args.workers
    return workload_config(args.config, **over)


# --------------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# -------------------------------------------------------------- reference arm --

def run_reference(args, wl, rank):
    """The CPU oracle (oracle/, plain single-threaded C) timed as it stands."""
    if rank != 0:
        return None
    import oracle

    from paper_2402_07529_b200.sizing import size_workload

    oracle.build()
    target = max(5.0, 150.0 / max(1, args.steps + args.warmup))
    # calibrate on a small prefix, then size the per-step sample to ~target seconds
    frac = 1.0
    cal = sample_workload(wl, 1 / 64)
    t_cal = oracle_step(oracle, cal, size_workload, args.gamma)
    trace(f"oracle calibration: {t_cal:.3f} s on d={cal.d}")
    est_full = t_cal * 64
    if est_full > target:
        frac = max(1 / 64, target / est_full)
    sub = sample_workload(wl, frac)
    times = []
    for s in range(args.warmup + args.steps):
        t = oracle_step(oracle, sub, size_workload, args.gamma)
        trace(f"oracle step {s}: {t:.2f} s on d={sub.d}")
        if s >= args.warmup:
            times.append(t)
    T = sum(times) / len(times)
    value = sub.d / T
    sample = (f"{sub.workers} workers x d={sub.d} ({frac:.3f} of {wl.name}'s d={wl.d}), "
              f"same density/structure/sizing rule; full pipeline per step")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": T * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": wl.name, "d": wl.d, "density": wl.density,
                       "workers": wl.workers, "structure": wl.structure},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, **host_cpu(),
                             "threads": "1 (the oracle is single-threaded C)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def host_cpu():
    """Host core count and CPU model of the box the oracle runs on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    if model is None:
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        except Exception:
            pass
    return {"host_cores": os.cpu_count(), "host_cpu": model or "unknown"}


def sample_workload(wl, frac):
    from lhc_inputs import Workload

    d = max(4096, int(wl.d * frac))
    kw = dict(wl.__dict__)
    kw["d"] = d
    return Workload(**kw)


def oracle_step(oracle, wl, size_workload, gamma):
    xs = [wl.dense(w) for w in range(wl.workers)]
    s = size_workload(wl.d, wl.density, wl.workers, gamma=gamma)
    p = oracle.params(wl.d, s.m, s.c, 3, 0, 1024, SEED)
    t0 = time.perf_counter()
    oracle.pipeline(p, xs)
    return time.perf_counter() - t0


# ------------------------------------------------------------------- our arm --

def trace(msg):
    if os.environ.get("LHC_BENCH_TRACE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


_OUT = None  # the JSON line's stream: the original stdout (fd 1 itself goes to stderr)


def emit(line):
    print(json.dumps(line), file=_OUT or sys.stdout, flush=True)


def main():
    global _OUT
    # rank 0 prints ONE JSON line on stdout: library banners (e.g. NCCL's version line)
    # and warnings written to fd 1 are sent to stderr instead
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    if os.environ.get("LHC_BENCH_TRACE"):
        import faulthandler

        faulthandler.dump_traceback_later(int(os.environ.get("LHC_BENCH_TRACE")), exit=True)
    wl = workload(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        line = run_reference(args, wl, rank)
        if line is not None:
            emit(line)
        return

    import torch
    import torch.distributed as dist

    import paper_2402_07529_b200 as lhc

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lhc.lib()

    from paper_2402_07529_b200.sizing import INDEX_BITMAP, smaller_index

    kb = {"bloom": 0, "bitmap": INDEX_BITMAP}.get(args.index)
    if kb is None:
        kb = smaller_index(wl.d, wl.density, wl.workers, gamma=args.gamma)
    nblocks = 0
    if args.blocks != "0":
        from paper_2402_07529_b200.sizing import size_blocked

        sz, nblocks = size_blocked(wl.d, wl.density, wl.workers, gamma=args.gamma, k_bloom=kb,
                                   L=args.L, cells_per_block=args.block_cells)
        if args.blocks != "auto":
            nblocks = int(args.blocks)
            S = max(1, -(-sz.c // (nblocks * 3 * args.L)))
            sz.c = nblocks * S * 3 * args.L
    else:
        sz = lhc.size_workload(wl.d, wl.density, wl.workers, gamma=args.gamma, k_bloom=kb, L=args.L)
    p = lhc.params(wl.d, sz.m, sz.c, 3, kb, args.L, SEED, nblocks)
    # candidate capacity: n_c concentrates within ~0.5 % of its expectation (runs of 64:
    # std ~ 64 sqrt(runs)); 5 % headroom, and stats.overflow would report a miss
    cap = min(wl.d, int(sz.n_cand_expected * 1.05) + 4096)
    my_workers = lhc.pipeline.owned_workers(wl.workers, rank, world)

    trace('inputs')
    # inputs resident in HBM (generated on the host with the shared seeded recipe)
    host = [wl.dense(w) for w in my_workers]
    xs = [torch.from_numpy(x).to(dev) for x in host]

    comm = None
    if args.decode == "auto":
        args.decode = "sharded" if world > 1 and args.comm != "nccl" else "replicated"
    sharded = args.decode == "sharded"
    if sharded:
        from paper_2402_07529_b200.sizing import shard_plan

        if args.comm == "nccl":
            raise SystemExit("--decode sharded needs --comm p2p or nvls")
        if args.blocks != "0":
            raise SystemExit("--blocks applies to the replicated decode")
        plan = shard_plan(wl.d, world, wl.density, wl.workers, gamma=args.gamma, k_bloom=kb)
        run = lhc.ShardedAllReduce(plan, seed=SEED, local_workers=len(xs),
                                   per_worker=args.per_worker, device=dev, comm=args.comm,
                                   deterministic=args.deterministic)
        p_dec = run.ps[rank]           # the shard this rank decodes
        G = plan.shards
    else:
        if world > 1 and args.comm == "p2p":
            comm = lhc.PeerComm(p)
        elif world > 1 and args.comm == "nvls":
            comm = lhc.NvlsComm(p)
        run = lhc.LosslessAllReduce(p, cap, local_workers=len(xs),
                                    per_worker=args.per_worker, comm=comm, device=dev,
                                    deterministic=args.deterministic)
        p_dec = p
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    nccl_state = {}

    def nccl_allreduce():
        # baseline exchange: NCCL sum of counters + all-gather of bitmaps + OR
        # (NCCL has no bitwise-OR reduction); torch ops, not the product path
        sk = run.sketch
        dist.all_reduce(sk.counters)
        if "g" not in nccl_state:
            nccl_state["g"] = torch.empty((world, sk.bitmap.numel()), dtype=torch.int32, device=dev)
        g = nccl_state["g"]
        dist.all_gather_into_tensor(g, sk.bitmap)
        out = g[0].clone()
        for r in range(1, world):
            out.bitwise_or_(g[r])
        sk.bitmap.copy_(out)

    # instrumented step: CUDA events around each phase on the launching stream
    phase_launches = None

    def step(ev=None, launches=None):
        def mark(name):
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                ev.append((name, e))

        def cnt(ph):
            n = lhc.last_launch_count()
            if launches is not None:
                launches[0] += n
            if phase_launches is not None:
                phase_launches[ph] = phase_launches.get(ph, 0) + n

        mark("start")
        if sharded:
            return sharded_step(mark, cnt)
        # all local workers' gradients in one compress launch (sketch_compress_batch)
        dst = run.worker_sketches if run.per_worker else [run.sketch] * len(xs)
        clr = run.worker_sketches if run.per_worker else [run.sketch]
        lhc.sketch_clear_batch(p, [t.bitmap for t in clr[::-1]], [t.counters for t in clr[::-1]])
        cnt("clear")
        mark("compress0")
        lhc.sketch_compress_batch(p, xs, [t.bitmap for t in dst], [t.counters for t in dst])
        cnt("compress")
        mark("compress1")
        if run.per_worker:
            lhc.aggregate(p, run.worker_sketches, run.sketch)
            cnt("aggregate")
        mark("aggregate")
        if world > 1:
            if comm is not None:
                comm.allreduce()
                cnt("allreduce")
            else:
                nccl_allreduce()
        mark("allreduce")
        dec = run.decoder
        dec.query(run.sketch)
        cnt("query")
        mark("query")
        dec.peel(run.sketch)
        cnt("peel")
        mark("peel")

    def sharded_step(mark, cnt):
        targets = run.worker_bufs if run.per_worker else [run.slots] * len(xs)
        clr = [sk for bufs in (run.worker_bufs if run.per_worker else [run.slots]) for sk in bufs]
        lhc.sketch_clear_batch(run.ps[0], [sk.bitmap for sk in clr[::-1]], [sk.counters for sk in clr[::-1]])
        cnt("clear")
        mark("compress0")
        # every (worker, shard) pair in one launch
        pairs = [(run.shard_input(x, q), sk, run.plan.shard_d(q))
                 for bufs, x in zip(targets, xs) for q, sk in enumerate(bufs)]
        lhc.sketch_compress_batch(run.ps[0], [a for a, _, _ in pairs], [b.bitmap for _, b, _ in pairs],
                                  [b.counters for _, b, _ in pairs], ds=[c for _, _, c in pairs])
        cnt("compress")
        mark("compress1")
        if run.per_worker:
            for q in range(G):
                lhc.sketch_aggregate(run.ps[q], [b[q].bitmap for b in run.worker_bufs],
                                     [b[q].counters for b in run.worker_bufs],
                                     run.slots[q].bitmap, run.slots[q].counters)
                cnt("aggregate")
        mark("aggregate")
        if world > 1:
            run.reduce_scatter()
            cnt("allreduce")
        mark("allreduce")
        dec = run.decoder
        dec.query(run.slots[rank])
        cnt("query")
        mark("query")
        dec.peel(run.slots[rank])
        cnt("peel")
        mark("peel")
        if world > 1:
            run.allgather()
            cnt("allgather")
        mark("allgather")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    trace('warmup')
    n_warm = max(3, args.warmup)  # timing rule: at least 3 untimed warm-up steps
    for _ in range(n_warm):
        step()
    barrier()

    trace('timed')
    # ---- timed region: K steps, per-step events, L2 flushed between steps ----
    clocks = ClockSampler(local_rank)
    phase = {"clear": 0.0, "compress": 0.0, "aggregate": 0.0, "allreduce": 0.0, "query": 0.0,
             "peel": 0.0,
             "allgather": 0.0}
    compress_launch_ms = []
    launches = [0]
    total_ms = 0.0

    def collect(ev):
        """Fold one step's (name, event) marks into the totals."""
        nonlocal total_ms
        st = ev[0][1]
        total_ms += st.elapsed_time(ev[-1][1])
        prev = st
        for name, e in ev[1:]:
            dt = prev.elapsed_time(e)
            if name == "compress1":
                compress_launch_ms.append(dt)
                phase["compress"] += dt
            elif name == "compress0":
                phase["clear"] += dt
            elif name in phase:
                phase[name] += dt
            prev = e

    graph = None
    if not args.no_graph:
        # the whole step as one CUDA graph: every kernel replayed without host launch
        # overhead (the cooperative kernels and the NVLink all-reduce are capturable;
        # the all-reduce keeps its barrier epoch on the device)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        cap_launches = [0]
        with torch.cuda.graph(graph, stream=side):
            stream = torch.cuda.current_stream()
            step(None, cap_launches)
        stream = torch.cuda.current_stream()
        stream.wait_stream(side)
        for _ in range(2):
            graph.replay()
        barrier()
    clocks.start()
    barrier()
    # (1) headline: K steps, device time per step from events around each step
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            step(None, launches)
        e1.record(stream)
        step_ms.append((e0, e1))
    barrier()
    if graph is not None:
        launches[0] = cap_launches[0] * args.steps
    # (2) per-kernel breakdown: K instrumented steps launched from the host, CUDA
    #     events between the kernels on the launching stream
    per_step = []
    for t in range(args.steps):
        flush.zero_()
        ev = []
        if t == 0:
            phase_launches = {}
        step(ev, None)
        if t == 0:
            launches_by_phase = dict(phase_launches)
            phase_launches = None
        per_step.append(ev)
    torch.cuda.synchronize()
    for ev in per_step:
        collect(ev)
    total_ms = sum(a.elapsed_time(b) for a, b in step_ms)

    barrier()
    ms = total_ms / args.steps
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    # keep the GPU loaded with untimed steps for ~0.6 s so the clock sampler
    # (nvidia-smi every 20 ms, started before the timed region) sees the step's
    # steady state, not only the few ms of the timed region; the count is the
    # same on every rank (the step holds collective barriers)
    for _ in range(max(1, min(4000, int(600.0 / max(ms_max, 1e-3))))):
        if graph is not None:
            graph.replay()
        else:
            step(None, None)
    barrier()
    clocks.stop()

    stats = run.decoder.read_stats()

    trace('e2e')
    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(x).pin_memory() for x in host]
        out_host = torch.empty(wl.d, dtype=torch.float32).pin_memory()
        out_dense = run.dense if sharded else run.decoder.dense
        dev_in = [torch.empty_like(x) for x in xs]
        h2d = sum(x.numel() * 4 for x in pinned)
        d2h = out_host.numel() * 4

        def e2e_step():
            for h, d_ in zip(pinned, dev_in):
                d_.copy_(h, non_blocking=True)
            run.step(dev_in)
            out_host.copy_(out_dense, non_blocking=True)

        for _ in range(2):
            e2e_step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n_e2e = max(3, min(args.steps, 10))
        e0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        barrier()
        e_ms = torch.tensor([e0.elapsed_time(e1) / n_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": wl.d / (float(e_ms.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": float(e_ms.item()),
               "path": f"pinned host x_w -> H2D -> {type(run).__name__}.step -> dense sum D2H"}
        if not np.isfinite(e2e["value"]):
            e2e = None

        # the same through the COO boundary (the gradients are sparse): pinned host
        # (idx, val) per worker -> H2D -> step_coo -> the aggregate's candidate list
        # (idx, val) and stats D2H (cap entries, no host sync inside).  Steps are
        # pipelined the way a training loop would run them: two engines alternate, the
        # H2D of step i+1 and the D2H of step i run on their own streams while step i
        # / i+1 computes (PCIe is full duplex); every step still moves all its bytes.
        coo_host = [wl.coo(w) for w in my_workers]
        if sharded:   # per-shard lists with shard-relative indices (split once on the host)
            coo_host = [c for i, v in coo_host for c in run.split_coo(i, v)]
        # all lists packed into one pinned host buffer (one H2D copy per step): for
        # list j, indices at [off_j, off_j + n_j), values at [tot + off_j, ...)
        lens = [len(i) for i, _ in coo_host]
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tot = int(offs[-1])
        pin_all = torch.empty(2 * tot, dtype=torch.int32).pin_memory()
        pa = pin_all.numpy()
        for j, (i, v) in enumerate(coo_host):
            pa[offs[j]:offs[j + 1]] = i.view(np.int32)
            pa[tot + offs[j]:tot + offs[j + 1]] = v.view(np.int32)
        pin_i = [pin_all[offs[j]:offs[j + 1]] for j in range(len(lens))]
        pin_v = [pin_all[tot + offs[j]:tot + offs[j + 1]].view(torch.float32) for j in range(len(lens))]
        if sharded:
            run_b = lhc.ShardedAllReduce(run.plan, seed=SEED, local_workers=len(xs),
                                         per_worker=args.per_worker, device=dev, comm=args.comm,
                                         deterministic=args.deterministic)
        else:
            comm_b = None
            if world > 1 and args.comm == "p2p":
                comm_b = lhc.PeerComm(p)
            elif world > 1 and args.comm == "nvls":
                comm_b = lhc.NvlsComm(p)
            run_b = lhc.LosslessAllReduce(p, cap, local_workers=len(xs),
                                          per_worker=args.per_worker, comm=comm_b, device=dev,
                                          deterministic=args.deterministic)
        engines = [run, run_b]
        ins, items_k, outs, dev_alls = [], [], [], []
        cap_ = run.decoder.cap
        for k in range(2):
            dev_all = torch.empty(2 * tot, dtype=torch.int32, device=dev)
            dev_i = [dev_all[offs[j]:offs[j + 1]] for j in range(len(lens))]
            dev_v = [dev_all[tot + offs[j]:tot + offs[j + 1]].view(torch.float32)
                     for j in range(len(lens))]
            dev_alls.append(dev_all)
            ins.append((dev_i, dev_v))
            pairs = list(zip(dev_i, dev_v))
            items_k.append([pairs[w * G:(w + 1) * G] for w in range(len(my_workers))]
                           if sharded else pairs)
            outs.append((torch.empty(cap_, dtype=torch.int32).pin_memory(),
                         torch.empty(cap_, dtype=torch.float32).pin_memory(),
                         torch.empty(32, dtype=torch.uint8).pin_memory()))
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        s_comp = stream
        ev = {n: [torch.cuda.Event() for _ in range(2)] for n in ("in", "comp", "out")}
        for k in range(2):
            for n in ev:
                ev[n][k].record(s_comp)

        def e2e_coo_step(i):
            k = i % 2
            s_in.wait_event(ev["comp"][k])            # step i-2 no longer reads ins[k]
            with torch.cuda.stream(s_in):
                dev_alls[k].copy_(pin_all, non_blocking=True)
                ev["in"][k].record(s_in)
            s_comp.wait_event(ev["in"][k])
            s_comp.wait_event(ev["out"][k])           # step i-2's results have left
            d = engines[k].step_coo(items_k[k], stream=s_comp)
            ev["comp"][k].record(s_comp)
            s_out.wait_event(ev["comp"][k])
            with torch.cuda.stream(s_out):
                oi, ov, ost = outs[k]
                oi.copy_(d.idx[:cap_], non_blocking=True)
                ov.copy_(d.val[:cap_], non_blocking=True)
                ost.copy_(d.stats, non_blocking=True)
                ev["out"][k].record(s_out)

        for i in range(2):
            e2e_coo_step(i)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        for i in range(n_e2e):
            e2e_coo_step(i)
        e1.record(s_out)
        torch.cuda.synchronize()
        barrier()
        c_ms = torch.tensor([e0.elapsed_time(e1) / n_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(c_ms, op=dist.ReduceOp.MAX)
        # the last step's results equal a serial step's (same inputs)
        st_b = lhc.read_stats(outs[(n_e2e - 1) % 2][2])
        # headline e2e: the sparse (COO) boundary, the natural host form of these
        # gradients; the dense-boundary measurement is kept beside it
        dense_e2e = e2e
        e2e = {"value": wl.d / (float(c_ms.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": sum(t.numel() * 4 for t in pin_i + pin_v),
               "d2h_bytes_per_step": 8 * cap_ + 32, "ms_per_step": float(c_ms.item()),
               "path": "pinned host COO (idx, val) per worker -> H2D -> "
                       f"{type(run).__name__}.step_coo -> candidate list (idx, val) + stats D2H"
                       + (" (own shard's list; every rank also holds the dense sum)"
                          if sharded else "")
                       + "; steps pipelined over 3 streams (H2D / compute / D2H), 2 engines",
               "decode_ok": bool(st_b["success"] and st_b["n_cand"] == stats["n_cand"]),
               "dense": dense_e2e}
        for eng in engines[1:]:
            if getattr(eng, "comm", None) is not None and hasattr(eng.comm, "close"):
                eng.comm.close()
            if hasattr(eng, "close"):
                eng.close()

    trace('roofline')
    # ---- roofline: every step of the path against its bound; the dominant one ----
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    nvl = 770.0  # measured peer copy per direction (B200_PROFILING.md)
    S = int(p.m) // 8 + 4 * int(p.c)
    n_c = stats["n_cand"]
    W_loc = len(xs)
    per_step_ms = {k: v / args.steps for k, v in phase.items()}
    avg_compress_ms = sum(compress_launch_ms) / max(1, len(compress_launch_ms))
    # algorithmic bytes per launch (Measurement) and launches per step
    if sharded:
        S_all = sum(int(q.m) // 8 + 4 * int(q.c) for q in run.ps)
        kern = {
            # one launch: every local worker's gradient into its G shard sketches
            "k_compress_dense": (W_loc * 4 * wl.d + (W_loc if run.per_worker else 1) * S_all, 1,
                                 avg_compress_ms, hbm, "hbm"),
            "k_aggregate": ((W_loc + 1) * S_all / G, G if run.per_worker else 0,
                            per_step_ms["aggregate"] / G, hbm, "hbm"),
            "k_reduce_scatter": ((world - 1) / world * S_all, 1 if world > 1 else 0,
                                 per_step_ms["allreduce"], nvl, "nvlink"),
            "k_query": (int(p_dec.m) // 8 + 4 * n_c, 1, per_step_ms["query"], hbm, "hbm"),
            "k_peel": (16 * int(p_dec.c) + 9 * n_c + 4 * int(p_dec.d), 1, per_step_ms["peel"],
                       hbm, "hbm"),
            # the own list to every peer (8 B per item)
            "k_allgather_decoded": (8 * n_c * (1 if args.comm == "nvls" else world - 1),
                                    1 if world > 1 else 0,
                                    per_step_ms["allgather"], nvl, "nvlink"),
        }
    else:
        kern = {
            # one launch: every local worker's gradient into its sketch (its own, or
            # the rank's one sketch when the workers are accumulated in place)
            "k_compress_dense": (W_loc * 4 * wl.d + (W_loc if run.per_worker else 1) * S, 1,
                                 avg_compress_ms, hbm, "hbm"),
            "k_aggregate": ((W_loc + 1) * S, 1 if run.per_worker else 0,
                            per_step_ms["aggregate"], hbm, "hbm"),
            # NVLink bytes out per rank: two-shot 2(G-1)/G S; NVLS (the switch pulls
            # every operand, one multicast store per slice) (1 + 1/G) S
            "k_allreduce": ((1 + 1 / world) * S if args.comm == "nvls" else 2 * (world - 1) / world * S,
                            1 if world > 1 and args.comm != "nccl" else 0,
                            per_step_ms["allreduce"], nvl, "nvlink"),
            "k_query": (int(p.m) // 8 + 4 * n_c, 1, per_step_ms["query"], hbm, "hbm"),
            # peel + finalize, and the dense output (zeroed, then the values at candidates)
            "k_peel": (16 * int(p.c) + 9 * n_c + 4 * wl.d, 1, per_step_ms["peel"], hbm, "hbm"),
        }
    n_clr = W_loc if run.per_worker else 1
    kern["k_clear"] = (n_clr * (S_all if sharded else S), 1, per_step_ms["clear"], hbm, "hbm")
    kernels = {}
    for name, (byts, nl, ms_l, peak, bound) in kern.items():
        if nl == 0 or ms_l <= 0:
            continue
        ach = byts / (ms_l * 1e-3) / 1e9
        phase_of = {"k_compress_dense": "compress", "k_aggregate": "aggregate", "k_allreduce": "allreduce",
                    "k_reduce_scatter": "allreduce", "k_query": "query", "k_peel": "peel",
                    "k_clear": "clear", "k_allgather_decoded": "allgather"}
        kernels[name] = {"bound": bound, "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "bytes_per_launch": int(byts),
                         "avg_launch_us": ms_l * 1e3, "launches_per_step": nl,
                         "us_per_step": ms_l * 1e3 * nl,
                         # kernels launched by the phase's API call (the peel phase also builds
                         # its state: k_pair_count/scan/scatter + k_build_cells when the state
                         # exceeds L2); its time is the whole phase's
                         "phase_launches": launches_by_phase.get(phase_of.get(name))}
    # the peel's own bound: L2 atomics (key inserts when the state is built in-kernel,
    # one claim per frontier entry, two updates per other cell of a peeled candidate)
    # against the measured ATOM.ADD.64-with-return peak (tools/atomic_peak.cu)
    if "k_peel" in kernels:
        pd = p_dec
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        insert = 3 * n_c if 16 * int(pd.c) <= l2 // 2 else 0
        n_atom = insert + stats.get("entries", 0) + 2 * (3 - 1) * stats["n_peeled"]
        t_peel = kernels["k_peel"]["avg_launch_us"] * 1e-6
        kernels["k_peel"]["l2_atomics"] = {
            "count": int(n_atom), "achieved": n_atom / t_peel / 1e9, "peak": 122.0,
            "unit": "G atomics/s", "frac": n_atom / t_peel / 1e9 / 122.0,
            "peak_source": "tools/atomic_peak.cu: random ATOM.ADD.64 with return, 64 MB footprint",
            "rounds": stats["rounds"], "entries": stats.get("entries", 0)}
    # measured DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum of
    # one `ncu --set full` capture of this workload at N = 1, profiles/traffic.json)
    traffic = {}
    tf = {}
    try:
        tf = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if world == 1 and not sharded and args.comm == "p2p":
            traffic = tf.get(wl.name + ("-bitmap" if kb == INDEX_BITMAP else ""), {})
    except Exception:
        pass
    for name in kernels:
        kernels[name]["traffic"] = traffic.get(name)
    # the query is bound by instruction issue, not bytes (ncu: IPC 2.0-2.5 of 4, DRAM
    # 2-7 %): warp instructions per launch (smsp__inst_executed.sum of the same capture,
    # profiles/traffic.json "inst") against 4 issues per SM per cycle at the max SM clock
    try:
        inst = tf.get("inst", {}).get(wl.name + ("-bitmap" if kb == INDEX_BITMAP else ""), {}) \
            if world == 1 and not sharded else {}
    except Exception:
        inst = {}
    if "k_query" in kernels and inst.get("k_query"):
        # a diagnostic, not a roofline: how busy the issue slots were (the kernel's own
        # instruction count from ncu over its time); the roofline is the HBM fraction
        cs = clocks.summary()
        mhz = cs.get("sm_max_mhz") or 1965.0
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        ipk = 4.0 * n_sm * mhz * 1e6 / 1e9  # G warp-instructions/s
        ach_i = inst["k_query"] / (kernels["k_query"]["avg_launch_us"] * 1e-6) / 1e9
        kernels["k_query"]["issue_utilisation"] = {
            "inst_per_launch": int(inst["k_query"]), "achieved": ach_i, "peak": ipk,
            "unit": "G warp-instructions/s", "frac": ach_i / ipk,
            "peak_source": f"{n_sm} SMs x 4 schedulers x {mhz:.0f} MHz (one issue per scheduler per cycle)"}
    dom = max(kernels, key=lambda k: kernels[k]["us_per_step"])
    roofline = dict(kernels[dom])
    roofline.update({"kernel": dom,
                     "peak_source": hbm_src if roofline["bound"] == "hbm" else
                     "B200_PROFILING.md measured peer copy 770 GB/s"})
    roofline = {k: roofline[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic",
                                         "kernel", "bytes_per_launch", "avg_launch_us",
                                         "peak_source")}
    if "l2_atomics" in kernels[dom]:
        roofline["l2_atomics"] = kernels[dom]["l2_atomics"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = run_reference(argparse.Namespace(steps=1, warmup=0, gamma=args.gamma, gpus=1), wl, 0)
        cpu = ref["cpu_baseline"] if ref else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": wl.d / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": n_warm, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl.name, "d": wl.d, "density": wl.density,
                       "workers": wl.workers, "structure": wl.structure, "law": wl.law,
                       "k": 3, "L": int(p.L), "m": int(p.m), "c": int(p.c), "gamma": args.gamma,
                       "blocks": int(p.blocks),
                       "index": "bitmap" if kb == INDEX_BITMAP else "bloom",
                       "sketch_bytes": int(p.m) // 8 + 4 * int(p.c),
                       "per_worker_sketches": run.per_worker,
                       "deterministic_decode": args.deterministic,
                       "decode": args.decode,
                       "comm": args.comm if world > 1 else "none",
                       "l2": "flushed (256 MB write) between timed steps, outside the events",
                       "cuda_graph": graph is not None,
                       "kernel_timing": "CUDA events between kernels in a second K-step pass "
                                        "launched from the host (same inputs, L2 flushed)"},
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches[0],
            "launches_per_step_by_phase": launches_by_phase,
            "clocks": clocks.summary(),
            "phases_ms_per_step": per_step_ms,
            "decode": stats,
        }
        emit(line)
    # a step whose decode overflowed its candidate capacity or stalled timed a
    # truncated peel: the line above records it, the exit code rejects it
    bad = torch.tensor([0 if stats["success"] and not stats["overflow"] else 1], device=dev)
    if world > 1:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    rc = 3 if int(bad.item()) else 0
    if rc:
        print(f"bench: decode failed (success={stats['success']}, overflow={stats['overflow']}); "
              "the timed steps are not a valid measurement", file=sys.stderr, flush=True)
    graph = None  # a captured graph may hold NCCL work: release it before the teardown
    torch.cuda.synchronize()
    if comm is not None:
        comm.close()
    if sharded:
        run.close()
    if world > 1:
        dist.barrier()
    _OUT.flush()
    sys.stderr.flush()
    os._exit(rc)  # no process-group teardown (it can hang on graph-captured NCCL work)


if __name__ == "__main__":
    main()
