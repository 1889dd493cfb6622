"""Write tests/golden/rowmap.json: the frozen hash / row-map table of reading R1-R2,
R4, R6, R7 ("The oracle freezes a golden table;
the GPU must reproduce it").

The paper gives no hash functions ("hashed to three signals ... and three
different indexes"), so the written spec of SURVEY.md §8c is the pin:

    mix64(z)  = SplitMix64 finalizer
    H(seed, dom, j, i) = mix64(seed ^ mix64(((dom<<56) | (j<<48) | i) + 0x9E3779B97F4A7C15))
    bias = H & (L-1);  sign = bit 16 of H ? -1 : +1;  row = j*S + ((H>>32) * S >> 32)

This script imports only ``oracle/`` (never the CUDA path).  It is run once; the
table it writes is committed, and ``tests/test_oracle.py`` checks the oracle
against it (so a later change to the oracle's packing, sign bit or row reduction
fails), while ``tests/test_gpu_parity.py::test_hash_rows_bit_exact`` checks the
CUDA hash kernel against the same file.

    python tools/make_golden_rowmap.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "rowmap.json")

# (seed, dom, j, i): SURVEY.md §8c's three sample values first, then probes of
# every packing field (dom, j, high bits of i) and seeds with high bits set
HASH_KEYS = [
    (0, 0, 0, 0), (0, 1, 0, 0), (0xDEADBEEF, 0, 2, 12345),
    (0, 0, 1, 0), (0, 0, 2, 0), (0, 1, 2, 0), (0, 0, 0, 1), (0, 0, 0, 1 << 20),
    (0, 0, 0, (1 << 40) + 3), (0, 0, 7, 99), (0x1DC0DE, 0, 0, 139648), (0x1DC0DE, 1, 2, 139648),
    (0xFFFFFFFFFFFFFFFF, 0, 1, 31249), (0x8000000000000000, 1, 0, 5), (0xDEADBEEF12345, 0, 2, 2999),
]

# Row-map tables: the configurations test_hash_rows_bit_exact launches on the GPU
# (d = 5e6, m = 3*L*1117, c = 3*L*733, seed 0xDEADBEEF12345, input rows 0..2999
# step 7), plus a paper-size partition count (VGG19 at gamma_s = 1.30: S_Y = 5218).
TABLES = [
    dict(d=5_000_000, L=L, S_Y=733, S_B=1117, seed=0xDEADBEEF12345, rows=list(range(0, 3000, 7)))
    for L in (32, 128, 1024)
] + [dict(d=143_000_000, L=1024, S_Y=5218, S_B=44956, seed=0x1DC0DE,
          rows=[0, 1, 2, 3, 1000, 65535, 65536, 139648])]


def main():
    oracle.build()
    hashes = [[s, dom, j, i, oracle.hash64(s, dom, j, i)] for (s, dom, j, i) in HASH_KEYS]
    tables = []
    for t in TABLES:
        p = oracle.params(t["d"], 3 * t["S_B"] * t["L"], 3 * t["S_Y"] * t["L"], 3, 3, t["L"], t["seed"])
        entries = []
        for dom in (0, 1):
            for i in t["rows"]:
                for j in range(3):
                    row, bias, sign = oracle.row_map(p, dom, j, i)
                    entries.append([dom, j, i, row, bias, sign])
        tables.append(dict(d=t["d"], L=t["L"], S_Y=t["S_Y"], S_B=t["S_B"], k=3, k_bloom=3,
                           seed=t["seed"], entries=entries))
    doc = {
        "what": "frozen hash / row-map table (readings R1, R2, R4, R6, R7; SURVEY.md §8c step 2)",
        "written_by": "tools/make_golden_rowmap.py (imports only oracle/)",
        "fields": {"hash": "[seed, dom, j, i, H]",
                   "entries": "[dom, j, i, row, bias, sign]; m = 3*S_B*L, c = 3*S_Y*L"},
        "hash": hashes,
        "tables": tables,
    }
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
        f.write("\n")
    print(f"wrote {OUT}: {len(hashes)} hashes, {sum(len(t['entries']) for t in tables)} row maps")


if __name__ == "__main__":
    main()
