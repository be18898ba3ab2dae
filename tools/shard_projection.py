"""Per-rank work of the N-GPU decomposition, measured on ONE GPU.

Runs every rank r < N of the row-sharded predictor (A's
nnz-balanced row shard, B replicated, rank r's share of the sample list) as a
*detached* shard -- world = N without a communicator, so no kernel waits on
another rank -- one after the other on cuda:0, and times each rank's step
with CUDA events on the predictor's stream (warm-up, L2-sized inputs).  The
max over ranks is what an N-GPU step costs before the one NCCL all-reduce of
40 bytes (not measurable with one GPU).  This is a load-balance and
strong-scaling projection, not a multi-GPU measurement.

  python tools/shard_projection.py [--config 5] [--ranks 1 2 4 8] [--steps 10]
prints one JSON object.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only-rank", type=int, default=-1, help="profile one rank of each world (ncu)")
    args = ap.parse_args()
    import torch
    from paper_2207_13848_b200 import gen
    from paper_2207_13848_b200.capi import DEVICE
    from paper_2207_13848_b200.spnnz import Predictor, SamplePolicy

    info = gen.CONFIGS[args.config]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        peak = 6650.0  # the profiling recipe's fallback
    a, b = gen.make_config(args.config)
    policy = SamplePolicy(info["fraction"], -1)
    out = {"config": info["name"], "nnz_A": a.nnz(), "kind": "detached shards on one GPU (projection)",
           "allreduce": "not included (one 40-byte NCCL all-reduce per step)", "per_world": {}}
    for world in args.ranks:
        per_rank = []
        for rank in range(world):
            if args.only_rank >= 0 and rank != min(args.only_rank, world - 1):
                continue
            P = Predictor(0, rank, world, None)
            P.load(a, None if b is a else b)
            P.synchronize()
            stream = torch.cuda.ExternalStream(P.stream_handle())
            dev_ceil = torch.empty(max(P.local_rows, 1), dtype=torch.int64, device="cuda")

            def step():
                return P.run_prediction(info["seed"], policy, ceil_out=dev_ceil, residency=DEVICE,
                                        want_real=False, want_samples=False)
            for _ in range(args.warmup):
                step()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            phase = np.zeros(5)
            torch.cuda.synchronize()
            for i in range(args.steps):  # timed as bench.py times: no per-phase events
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            P.set_profiling(True)  # then the phases, the same number of steps
            for i in range(args.steps):
                step()
                t, _ = P.last_timings()
                phase += np.array([t[k] for k in ("flop", "sample", "symbolic", "allreduce", "predict")])
            torch.cuda.synchronize()
            P.set_profiling(False)
            ms = float(np.mean([s.elapsed_time(e) for s, e in ev]))
            # the FLOP pass of this rank against the HBM roofline (bench.py's
            # algorithmic bytes for its shard, measured copy peak)
            nnz_local = int(a.rpt[P.row_hi] - a.rpt[P.row_lo])
            fbytes = 8 * (P.local_rows + 1) + 4 * nnz_local + 8 * (b.rows + 1) + 8 * P.local_rows
            flop_ms = phase[0] / args.steps
            per_rank.append({"rank": rank, "rows": P.local_rows, "nnz": nnz_local, "ms": ms,
                             "flop_pass_GBps": fbytes / (flop_ms * 1e-3) / 1e9 if flop_ms else None,
                             "flop_pass_hbm_frac": fbytes / (flop_ms * 1e-3) / 1e9 / peak if flop_ms else None,
                             "phases_ms": dict(zip(("flop", "sample", "symbolic", "allreduce", "predict"),
                                                   (phase / args.steps).round(4).tolist()))})
            P.close()
            del dev_ceil
            torch.cuda.empty_cache()
        mx = max(r["ms"] for r in per_rank)
        mean = float(np.mean([r["ms"] for r in per_rank]))
        out["per_world"][str(world)] = {"max_ms": mx, "mean_ms": mean, "imbalance": mx / mean,
                                        "projected_A_nnz_per_s": a.nnz() / (mx * 1e-3),
                                        "flop_pass_hbm_frac_mean": float(np.mean(
                                            [r["flop_pass_hbm_frac"] or 0 for r in per_rank])),
                                        "ranks": per_rank}
    base = out["per_world"].get("1") if args.only_rank < 0 else None
    if base:
        for w, d in out["per_world"].items():
            d["projected_speedup"] = base["max_ms"] / d["max_ms"]
            d["projected_efficiency"] = d["projected_speedup"] / int(w)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
