"""The C++ API of the drop-in boundary (csrc/include/ustats/*.hpp, exported
from libustats_b200.so): a C++ caller compiles and links against it, the
reference's own callers of the path (hoif.cpp, dcov.cpp, motifs.cpp) relink
unchanged, and on the GPU the caller reproduces the reference's engine test
and its hoif_tau."""
import os
import shutil
import subprocess
from math import comb
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
INC = ROOT / "paper_2508_12627_b200" / "csrc" / "include"
LIBDIR = ROOT / "paper_2508_12627_b200"
REF_SRC = Path("/root/reference/proj/src")


def _gxx():
    return shutil.which("g++") or "g++"


def _build_caller(tmp_path):
    import paper_2508_12627_b200 as us
    us.lib()  # built
    exe = tmp_path / "engine_api"
    subprocess.run([_gxx(), "-std=c++20", "-O1", f"-I{INC}", str(ROOT / "tests" / "cpp" / "engine_api.cpp"), "-o",
                    str(exe), f"-L{LIBDIR}", "-lustats_b200", f"-Wl,-rpath,{LIBDIR}"], check=True, capture_output=True)
    return exe


def test_cpp_caller_links(tmp_path):
    exe = _build_caller(tmp_path)
    assert exe.exists()
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(LIBDIR / "libustats_b200.so")], capture_output=True,
                          text=True, check=True).stdout
    for name in ("ustats::u_statistic(", "ustats::v_statistic(", "ustats::restricted_v(", "ustats::hoif_tau(",
                 "ustats::einsum(", "ustats::optimize_order(", "ustats::SparsifiedPartitionStream::",
                 "ustats::tensorize(", "ustats::fail("):
        assert name in syms, name


@pytest.mark.skipif(not REF_SRC.is_dir(), reason="reference sources not present (GPU box)")
def test_reference_callers_relink_unchanged(tmp_path):
    # the reference's callers of u_statistic, compiled from their own sources
    # against our headers, link against libustats_b200.so with nothing undefined
    objs = []
    for f in ("hoif", "dcov", "motifs"):
        o = tmp_path / f"{f}.o"
        subprocess.run([_gxx(), "-std=c++20", "-O1", "-fPIC", f"-I{INC}", "-I/root/reference/proj/include", "-c",
                        str(REF_SRC / f"{f}.cpp"), "-o", str(o)], check=True, capture_output=True)
        objs.append(str(o))
    subprocess.run([_gxx(), "-shared", "-o", str(tmp_path / "libcallers.so"), *objs, f"-L{LIBDIR}", "-lustats_b200",
                    "-Wl,--no-undefined"], check=True, capture_output=True)


@pytest.mark.gpu
def test_cpp_caller_runs_reference_cases(tmp_path):
    from oracle import ref as REF
    exe = _build_caller(tmp_path)
    rng = np.random.default_rng(7)
    n, d, m, k = 300, 6, 4, 3
    x = rng.normal(size=(n, d))
    f = tmp_path / "sample.bin"
    f.write_bytes(np.array([n, d], dtype=np.int64).tobytes() + x.tobytes())
    out = subprocess.run([str(exe), str(f), str(m), str(k)], capture_output=True, text=True, check=True).stdout
    lines = dict(line.split(" ", 1) for line in out.strip().splitlines())
    vals = dict(kv.split("=") for kv in lines["prod2"].split())
    # test_engine.cpp:106-116: exact small integers
    assert float(vals["V"]) == 36.0 and float(vals["U"]) == 22.0
    assert float(vals["coarsest"]) == 14.0 and float(vals["finest"]) == 36.0
    assert lines["error"] == "SampleTooSmall"
    tau = float(lines["hoif"].split()[0])
    if REF.available():
        want = REF.hoif_tau(m, k, x)
        assert abs(tau - want) <= 1e-9 * _hoif_scale(m, k, x)


def _hoif_scale(m, k, x):
    # the largest weighted chain statistic of the expansion (cancellation scale)
    import paper_2508_12627_b200 as us
    n = x.shape[0]
    u = {o: us.u_statistic(f"hoif:{o}:{k}", x) for o in range(2, m + 1)}
    best = 0.0
    for j in range(2, m + 1):
        for l in range(j - 1):
            w = 1.0
            for i in range(l):
                w /= n - i
            best = max(best, abs(comb(j - 2, l) * w * u[l + 2]))
    return best


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,k", [(256, 4, 3), (512, 5, 2), (300, 2, 4), (257, 6, 3)])
def test_hoif_tau_device_matches_reference(n, m, k):
    # us_hoif_tau: device tensorization, chain orders in one program, long
    # double combination == the reference's hoif_tau (hoif.cpp:74-100)
    from oracle import ref as REF
    import paper_2508_12627_b200 as us
    if not REF.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(n + m + k)
    x = rng.normal(size=(n, 2 + k + 1))
    got, st = us.hoif_tau(m, k, x, with_stats=True)
    want = REF.hoif_tau(m, k, x)
    assert abs(got - want) <= 1e-9 * _hoif_scale(m, k, x), (got, want)
    assert st["kernel_launches"] > 0
    import torch
    got_dev = us.hoif_tau(m, k, torch.from_numpy(x).cuda())
    assert got_dev == got


def test_hoif_tau_argument_errors():
    import paper_2508_12627_b200 as us
    x = np.zeros((10, 5))
    for args, code in [((1, 2, x), "InvalidArgument"), ((3, 0, x), "InvalidArgument"), ((3, 4, x), "InvalidArgument"),
                       ((12, 2, x), "SampleTooSmall")]:
        with pytest.raises(us.UStatsError) as e:
            us.hoif_tau(*args)
        assert e.value.code == code
