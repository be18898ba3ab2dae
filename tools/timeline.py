"""Per-stream end times of the predictor's call (SPNNZ_DEBUG_TIMELINE=1,
eager calls): python tools/timeline.py [config] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SPNNZ_DEBUG_TIMELINE"] = "1"
os.environ["SPNNZ_GRAPH"] = "0"
from paper_2207_13848_b200 import gen  # noqa: E402
from paper_2207_13848_b200.spnnz import Predictor, SamplePolicy  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
info = gen.CONFIGS[cfg]
a, b = gen.make_config(cfg)
P = Predictor(0)
P.load(a, None if b is a else b)
for _ in range(steps):
    P.run_prediction(info["seed"], SamplePolicy(info["fraction"], -1), want_real=False, want_samples=False)
P.close()
