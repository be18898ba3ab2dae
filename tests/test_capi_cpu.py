"""CPU: the C-ABI library loads, exports every symbol include/spnnz_gpu/capi.h
declares, and its host-only logic (shard partition, sample count, scalar
estimators, error mapping) behaves like the reference.  No kernel launches."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2207_13848_b200 import capi, gen
from paper_2207_13848_b200.capi import lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spnnz_gpu", "capi.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spnnz_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = lib()
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(capi.EXPORTED)


def test_abi_version():
    assert lib().spnnz_gpu_abi_version() == 1


def test_so_is_sm100a():
    # the product kernels are compiled for sm_100a only (no PTX/other archs)
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_create_without_gpu_fails_loudly():
    import shutil
    import subprocess
    if shutil.which("nvidia-smi") and subprocess.run(["nvidia-smi", "-L"], capture_output=True).returncode == 0:
        pytest.skip("a GPU is present")
    ctx = ctypes.c_void_p()
    rc = lib().spnnz_gpu_create(0, 0, 1, None, ctypes.byref(ctx))
    assert rc == capi.ECUDA
    assert b"CUDA" in lib().spnnz_gpu_last_error() or b"device" in lib().spnnz_gpu_last_error()


def partition(rpt, world):
    out = np.zeros(world + 1, np.int32)
    capi.check(lib().spnnz_gpu_partition_rows(rpt.ctypes.data, len(rpt) - 1, world, out.ctypes.data))
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_rows_is_work_balanced(world):
    a = gen.rmat(14, 16 << 14, 0.57, 0.19, 0.19, 9)
    b = partition(a.rpt, world)
    assert b[0] == 0 and b[-1] == a.rows and (np.diff(b) >= 0).all()
    work = a.nnz() + a.rows
    w = a.rpt + np.arange(a.rows + 1)  # work of rows [0, i): entries + rows
    for r in range(1, world):
        # first row whose work reaches r*(nnz + rows)/world
        t = work // world * r + work % world * r // world
        assert w[b[r]] >= t and (b[r] == 0 or w[b[r] - 1] < t)


def test_partition_edge_cases():
    empty = np.zeros(1, np.int64)
    assert partition(empty, 4).tolist() == [0, 0, 0, 0, 0]
    one = np.array([0, 5], np.int64)
    assert partition(one, 2).tolist() == [0, 1, 1]


def test_sample_count_query_needs_no_gpu():
    from paper_2207_13848_b200.spnnz import SamplePolicy, plan_size
    for m, n in [(1000, 3), (1000000, 300), (100, 1), (1, 1), (100000, 300), (13514, 41)]:
        assert plan_size(m, SamplePolicy())[0] == n  # test_predict.cpp:26-33
    assert plan_size(1000, SamplePolicy(0.01, 50))[0] == 10
    assert plan_size(1 << 24, SamplePolicy(0.001, -1)) == (16778, 16778 / (1 << 24))
    with pytest.raises(ValueError):
        plan_size(0, SamplePolicy())


def test_estimators_match_reference_examples():
    from paper_2207_13848_b200 import spnnz
    st = spnnz.SampleStats(300, 100, 3.0)
    pp = spnnz.predict_proposed(st, 30000)  # test_predict.cpp:74-81
    assert pp.predicted_cr == 3.0 and pp.z2_star == 10000.0
    pp = spnnz.predict_proposed(spnnz.SampleStats(), 12345)  # :83-88
    assert pp.predicted_cr == 1.0 and pp.z2_star == 12345.0
    plan = spnnz.SamplePlan(p=0.003)
    assert math.isclose(spnnz.predict_reference(spnnz.SampleStats(sampled_nnz=30), plan), 10000.0)
    with pytest.raises(ValueError):
        spnnz.predict_reference(spnnz.SampleStats(), spnnz.SamplePlan(p=0.0))
    e = spnnz.error_report(125.0, 1000.0 / 130.0 * 12.5, 130, 100, 1000, 0.1)  # :114-125
    assert math.isclose(e.eps1, 0.25, rel_tol=1e-12) and abs(abs(e.eps2) * 100 - 3.85) < 0.005
    with pytest.raises(ValueError):
        spnnz.error_report(1.0, 1.0, 1, 0, 10, 0.1)
    assert lib().spnnz_sampled_cr(0, 5) == 1.0 and lib().spnnz_sampled_cr(6, 3) == 2.0


def test_estimators_bitwise_equal_oracle(oracle):
    """The host tail and the oracle evaluate identical IEEE expressions."""
    from paper_2207_13848_b200 import spnnz
    rng = np.random.default_rng(7)
    for _ in range(2000):
        F = int(rng.integers(1, 2**62))
        f = int(rng.integers(1, 2**40))
        z = int(rng.integers(1, f + 1))
        p = float(rng.random()) + 1e-9
        z1, z2, cr = oracle.estimators(f, z, F, p)
        pp = spnnz.predict_proposed(spnnz.SampleStats(f, z), F)
        assert pp.z2_star == z2 and pp.predicted_cr == cr
        assert spnnz.predict_reference(spnnz.SampleStats(f, z), spnnz.SamplePlan(p=p)) == z1


def test_exhaustive_plan():
    from paper_2207_13848_b200 import spnnz
    p = spnnz.exhaustive_plan(5)
    assert p.sample_rows.tolist() == [0, 1, 2, 3, 4] and p.p == 1.0
    with pytest.raises(ValueError):
        spnnz.exhaustive_plan(0)


def test_cpp_header_accepts_reference_csr(tmp_path):
    """The C++ mirror compiles against the reference's own spnnz::CsrMatrix
    (drop-in: callers keep their matrix type).  Needs /root/reference."""
    import subprocess
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers not present")
    src = tmp_path / "dropin_ref.cpp"
    src.write_text(
        '#include "spnnz/csr.hpp"\n#include "spnnz_gpu/spnnz_gpu.hpp"\n'
        "int main() { spnnz::CsrMatrix a; a.rows = a.cols = 1; a.rpt = {0, 1}; a.col = {0};\n"
        "  auto p = spnnz::gpu::compute_flop(a, a);\n"
        "  auto r = spnnz::gpu::run_prediction(a, a, 1, {0.5, 10});\n"
        "  auto e = spnnz::gpu::exact_symbolic(a, a, p);\n"
        "  return int(p.total_flop + r.total_flop + e.total_nnz) == 0; }\n")
    out = tmp_path / "dropin_ref"
    r = subprocess.run(["g++", "-std=c++20", "-I", ref_inc, "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(out), "-L", os.path.dirname(capi.LIB_PATH),
                        "-lspnnz_gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_nccl_id_before_torch_import_keeps_torch_importable():
    """Creating an NCCL id loads NCCL before torch: it must be the NCCL torch
    itself uses (or bound locally), so a later `import torch` still resolves
    its newer NCCL symbols."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2207_13848_b200.spnnz import Predictor\n"
            "assert len(Predictor.nccl_unique_id()) == 128\n"
            "import torch\n"
            "print('ok', torch.__version__)\n") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
