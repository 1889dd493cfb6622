"""Compress bandwidth probe on one GPU (VGG19 size by default): the batched dense
compress of the 8 workers into one sketch, against the same launch on all-zero
inputs (no reductions: the input stream alone) and torch's read of the same bytes.

    [LHC_LIB=...] python tools/compress_probe.py [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2402_07529_b200 as lhc  # noqa: E402
from paper_2402_07529_b200 import _lib as L  # noqa: E402
from lhc_inputs import config  # noqa: E402


def timed(fn, flush, reps=10):
    ts = []
    for _ in range(reps):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "vgg"
    dev = torch.device("cuda", 0)
    torch.zeros(1, device=dev)
    if os.environ.get("PERSIST"):
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
        v = ctypes.c_int(0)
        rt.cudaDeviceGetAttribute(ctypes.byref(v), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
        frac = float(os.environ["PERSIST"])
        err = rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(int(v.value * frac)))  # cudaLimitPersistingL2CacheSize
        print(f"persisting L2 limit {v.value * frac / 2**20:.1f} MB (max {v.value / 2**20:.1f}), err {err}")
    wl = config(name, law="gauss")
    s = lhc.size_workload(wl.d, wl.density, wl.workers)
    p = lhc.params(wl.d, s.m, s.c, 3, 0, 1024, 0x1DC0DE)
    xs = [torch.from_numpy(wl.dense(w)).to(dev) for w in range(wl.workers)]
    zs = [torch.zeros_like(x) for x in xs]
    sk = lhc.Sketch(p, device=dev)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)  # 256 MB
    n = len(xs)
    in_bytes = sum(x.numel() * 4 for x in xs)
    sk_bytes = sk.nbytes

    def comp(inputs):
        return lambda: L.sketch_compress_batch(p, inputs, [sk.bitmap] * n, [sk.counters] * n)

    # the same reductions into a sketch that fits in L2 (16 MB of counters, 4 MB index)
    ps = lhc.params(wl.d, 3 * 1024 * 10240, 3 * 1024 * 1360, 3, 0, 1024, 0x1DC0DE)
    sks = lhc.Sketch(ps, device=dev)

    def comp_small():
        return L.sketch_compress_batch(ps, xs, [sks.bitmap] * n, [sks.counters] * n)

    for nm, fn in [("compress", comp(xs)), ("compress(zeros)", comp(zs)),
                   ("compress(L2 sketch)", comp_small),
                   ("torch sum (read)", lambda: [x.sum() for x in xs]),
                   ("sketch clear", lambda: sk.clear())]:
        for _ in range(3):
            fn()
        us = timed(fn, flush)
        b = in_bytes + (sk_bytes if nm.startswith("compress") else 0)
        if nm == "sketch clear":
            b = sk_bytes
        print(f"{name} {nm:18s} {us:8.1f} us  {b / us / 1e3:7.1f} GB/s")


if __name__ == "__main__":
    main()
