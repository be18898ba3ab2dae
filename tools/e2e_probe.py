"""Timing probe of the end-to-end path pieces (config 5): H2D load alone,
load + prediction, prediction alone -- wall clock around synchronized calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2207_13848_b200 import gen
from paper_2207_13848_b200.capi import HOST
from paper_2207_13848_b200.spnnz import Predictor, SamplePolicy

a, _ = gen.make_config(5)
pin = lambda x: torch.from_numpy(x).pin_memory().numpy()  # noqa: E731
ha = type(a)(a.rows, a.cols, pin(a.rpt), pin(a.col))
P = Predictor(0)
host_ceil = torch.empty(a.rows, dtype=torch.int64).pin_memory().numpy()
pol = SamplePolicy(0.001, -1)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    P.synchronize()
    s = time.perf_counter()
    for _ in range(n):
        fn()
        P.synchronize()
    return (time.perf_counter() - s) / n * 1e3


print("load only      %.2f ms" % t(lambda: P.load(ha, None, residency=HOST)))
print("load + predict %.2f ms" % t(lambda: (P.load(ha, None, residency=HOST),
                                            P.run_prediction(5, pol, ceil_out=host_ceil, residency=HOST,
                                                             want_real=False, want_samples=False))))
print("predict (host out) %.2f ms" % t(lambda: P.run_prediction(5, pol, ceil_out=host_ceil, residency=HOST,
                                                                 want_real=False, want_samples=False)))
