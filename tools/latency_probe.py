"""Wall-clock latency per call of the small-problem entry points (host
overhead + graph replay), for the harness's tasks: python tools/latency_probe.py"""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_13848_b200 import gen  # noqa: E402
from paper_2207_13848_b200.capi import HOST, Report, check, lib  # noqa: E402
from paper_2207_13848_b200.spnnz import Predictor, SamplePolicy  # noqa: E402


def per_call(fn, n=200):
    for _ in range(5):
        fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n * 1e6


def main():
    L = lib()
    for name, (a, b) in {"cfg1": gen.make_config(1), "synth150k": (gen.synthetic("uniform", 150000, 150000, 8, 71),) * 2}.items():
        P = Predictor(0)
        P.load(a, None if b is a else b)
        ctx = P.ctx
        t, m = ctypes.c_int64(), ctypes.c_int64()
        flop = lambda: check(L.spnnz_gpu_compute_flop(ctx, None, HOST, ctypes.byref(t), ctypes.byref(m)))  # noqa: E731
        z = ctypes.c_int64()
        exact = lambda: check(L.spnnz_gpu_exact_symbolic(ctx, None, HOST, ctypes.byref(z)))  # noqa: E731
        rep = Report()
        pred = lambda: check(L.spnnz_gpu_predict_sampled(ctx, 97, 0.003, 300, ctypes.byref(rep), None))  # noqa: E731
        run = lambda: check(L.spnnz_gpu_run_prediction(ctx, 97, 0.003, 300, ctypes.byref(rep), None, None, None, HOST))  # noqa: E731
        out = {}
        for k, fn in (("compute_flop", flop), ("exact_symbolic", exact), ("predict_sampled", pred),
                      ("run_prediction", run)):
            if k == "predict_sampled":
                flop()
            out[k] = round(per_call(fn), 1)
            n = ctypes.c_int64()
            L.spnnz_gpu_last_timings(ctx, None, ctypes.byref(n))
            out[k + "_launches"] = n.value
        print(name, out)
        P.close()


if __name__ == "__main__":
    main()
