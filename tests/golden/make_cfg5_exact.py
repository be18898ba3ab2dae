"""Pins config 5's exact per-row NNZ to the REFERENCE ITSELF (oracle/_ref).

`make_golden.py` skips the exact pass on config 5 (F = 1.3e11 products, about
an hour of CPU).  This script runs the reference's own
`spnnz::exact_symbolic` (symbolic.hpp:94-118) over config 5 in row slices:
every slice is a row range of A handed to the unmodified reference
function with threads = 1, and the slices are scheduled dynamically over all
host threads (the reference's own `parallel_blocks` gives each thread one
contiguous block, parallel.hpp:30-41, which puts every R-MAT hub row on
thread 0).  Row i of a slice is row lo + i of A and the reference computes
each row independently (symbolic.hpp:104-113), so the concatenation is the
reference's exact_symbolic of the whole matrix.

Writes into tests/golden/configs.json["5"]:
  Z, exact_nnz (sha256[:32] of the int64 per-row array, same digest as the
  other configs), exact_nnz_blocks (the same digest per 2^20-row block, to
  localise a mismatch) and per mode the reference's error_report.
The full array is also cached (not committed) at build/cfg5_exact_nnz.npy.

Run here, where /root/reference exists:  python tests/golden/make_cfg5_exact.py
(`... make_cfg5_exact.py 2` re-derives config 2 the same way and checks it
against make_golden.py's whole-matrix run: the slicing self-check.)
"""
from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference  # noqa: E402
from paper_2207_13848_b200 import gen  # noqa: E402
from tests.golden.make_golden import digest  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
BLOCK = 1 << 20


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
    if not Reference.available():
        sys.exit("oracle/_ref not built: run `make -C oracle` where /root/reference exists")
    path = os.path.join(OUT, "configs.json")
    recs = json.load(open(path))
    rec = recs[cfg]
    t0 = time.time()
    a, b = gen.make_config(int(cfg))
    assert b is a
    assert digest(a.col) == rec["input"]["a_col"] and digest(a.rpt) == rec["input"]["a_rpt"]
    print(f"generated config {cfg} in {time.time() - t0:.0f}s", flush=True)
    R = Reference(threads=1)
    hb = R.matrix(b)
    flop, F, mx, prof = R.compute_flop(hb, hb, a.rows, keep_profile=True)
    R.L.ref_profile_free(prof)
    assert F == rec["F"] and digest(flop) == rec["flop"]
    M = a.rows
    # slices of ~F/4096 products (a hub row is its own slice)
    csum = np.cumsum(flop)
    target = max(1, F // 4096)
    bounds = [0]
    while bounds[-1] < M:
        lo = bounds[-1]
        base = csum[lo - 1] if lo else 0
        hi = int(np.searchsorted(csum, base + target, side="left")) + 1
        bounds.append(min(M, max(lo + 1, hi)))
    slices = list(zip(bounds[:-1], bounds[1:]))
    slices.sort(key=lambda s: -(csum[s[1] - 1] - (csum[s[0] - 1] if s[0] else 0)))
    print(f"{len(slices)} slices", flush=True)
    nnz = np.zeros(M, np.int64)
    lock = threading.Lock()
    nxt = [0]
    done = [0]

    def worker():
        Rw = Reference(threads=1)
        while True:
            with lock:
                if nxt[0] >= len(slices):
                    return
                lo, hi = slices[nxt[0]]
                nxt[0] += 1
            rpt = a.rpt[lo:hi + 1] - a.rpt[lo]
            col = a.col[a.rpt[lo]:a.rpt[hi]]
            ha = Rw.L.ref_matrix_new(hi - lo, a.cols, rpt.ctypes.data, col.ctypes.data)
            _, _, _, p = Rw.compute_flop(ha, hb, hi - lo, keep_profile=True)
            out, _ = Rw.exact_symbolic(ha, hb, p, hi - lo)
            Rw.L.ref_profile_free(p)
            Rw.free_matrix(ha)
            nnz[lo:hi] = out
            with lock:
                done[0] += 1
                if done[0] % 256 == 0:
                    print(f"  {done[0]}/{len(slices)} slices, {time.time() - t0:.0f}s", flush=True)

    nthreads = int(os.environ.get("SPNNZ_GOLDEN_THREADS", os.cpu_count() or 1))
    ths = [threading.Thread(target=worker) for _ in range(nthreads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    Z = int(nnz.sum())
    if cfg != "5":  # self-check against the whole-matrix reference run of make_golden.py
        assert Z == rec["Z"] and digest(nnz) == rec["exact_nnz"], (Z, rec["Z"])
        print(f"config {cfg}: slice-wise reference exact pass matches ({Z})")
        return
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    np.save(os.path.join(ROOT, "build", "cfg5_exact_nnz.npy"), nnz)
    rec["Z"] = Z
    rec["exact_nnz"] = digest(nnz)
    rec["exact_nnz_blocks"] = [digest(nnz[i:i + BLOCK]) for i in range(0, M, BLOCK)]
    rec["exact_seconds"] = time.time() - t0
    rec["exact_method"] = ("reference spnnz::exact_symbolic (oracle/_ref) over row slices of A, "
                           "threads=1 per slice, slices scheduled over all host threads")
    for label in rec["modes"]:
        r = rec["modes"][label]["report"]
        rec["modes"][label]["errors"] = R.error_report(r["z1_star"], r["z2_star"],
                                                       r["sampled_flop"], Z, F, r["p"])
    recs["5"] = rec
    with open(path, "w") as f:
        json.dump(recs, f, indent=1)
    print(f"config 5: Z = {Z} in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
