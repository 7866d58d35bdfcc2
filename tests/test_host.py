"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares, the host-side API validates like the reference, the bench
CPU-baseline estimator is consistent, and the build is sm_100a."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    txt = (ROOT / "include" / "tlrb200.h").read_text()
    return sorted(set(re.findall(r"\b(tlrb_[a-z_]+)\s*\(", txt)))


def test_library_exports_header_symbols(tb):
    from paper_1804_09137_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    declared = {name for name, _, _ in _lib.SIGNATURES}
    assert declared == set(syms)


def test_library_is_sm100a():
    so = ROOT / "paper_1804_09137_b200" / "libtlrb200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_dmma_in_sass():
    so = ROOT / "paper_1804_09137_b200" / "libtlrb200.so"
    out = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    # the FP64 GEMM issues mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; every tile
    # configuration of the template must carry it
    secs = [f.split("Function :", 1)[0] for f in out.split("dgemm_tiles_kernel")[1:]]
    assert len(secs) >= 5
    for sec in secs:
        assert sec.count("DMMA") >= 16


def test_generate_locations_matches_oracle(tb):
    from oracle import tlr_oracle as orc
    for n, seed in [(1, 0), (7, 3), (1600, 0), (10001, 5)]:
        np.testing.assert_array_equal(tb.generate_locations(n, seed).coords,
                                      orc.generate_locations(n, seed))


def test_param_validation(tb):
    with pytest.raises(ValueError):
        tb.MaternParams(0.0, 0.1, 0.5)
    with pytest.raises(ValueError):
        tb.MaternParams(1.0, 0.1, 5.5)
    with pytest.raises(ValueError):
        tb.MaternParams(1.0, 0.1, 0.5, -1.0)
    with pytest.raises(ValueError):
        tb.LikelihoodConfig(mode="tlr")
    with pytest.raises(ValueError):
        tb.LikelihoodConfig(mode="tlr", accuracy=1.5)
    with pytest.raises(ValueError):
        tb.LocationSet(np.array([[0.0, 0.0], [0.0, 0.0]]))
    with pytest.raises(ValueError):
        tb.LocationSet(np.zeros((3, 3)))


def test_shape_error_before_device(tb):
    locs = tb.generate_locations(10, 0)
    with pytest.raises(ValueError):
        tb.log_likelihood(locs, np.zeros(9), tb.MaternParams(1.0, 0.1, 0.5))


def test_tile_size_defaults(tb):
    assert tb.LikelihoodConfig().tile_size() == 200
    assert tb.LikelihoodConfig(mode="tlr", accuracy=1e-9).tile_size() == 400
    assert tb.LikelihoodConfig(nb=77).tile_size() == 77


def test_cpu_baseline_estimator_runs():
    from oracle import cpu_baseline as cb
    from oracle import tlr_oracle as orc
    xy = orc.generate_locations(600, 0)
    z = np.random.default_rng(0).standard_normal(600)
    est, desc = cb.estimate_eval_seconds(xy, z, (1.0, 0.1, 0.5), 100, 1e-7)
    assert est > 0 and "recompressions" in desc
    est_d, _ = cb.estimate_eval_seconds(xy, z, (1.0, 0.1, 0.5), 100, None)
    assert est_d > 0


def test_no_oracle_import_in_product():
    pkg = ROOT / "paper_1804_09137_b200"
    for p in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*")):
        assert "oracle" not in p.read_text().replace("oracle-free", ""), p


def test_no_forbidden_batched_copies():
    # the batched-copy driver calls fault on this driver (B200_PROFILING.md)
    bad = ["Memcpy" + "Batch", "Memcpy3D" + "Batch"]
    for p in (ROOT / "paper_1804_09137_b200" / "csrc").glob("*"):
        assert not any(b in p.read_text() for b in bad), p


def test_recorded_bench_line_contract():
    """The committed bench line (profiles/r02_bench_c3.json, produced on a
    B200 by bench.py on the C3 headline config) carries every key of the
    driver contract."""
    import json
    from conftest import ROOT

    d = json.loads((ROOT / "profiles" / "r02_bench_c3.json").read_text().strip().splitlines()[-1])
    assert d["config"]["workload"].startswith("C3 n=62500")
    assert d["roofline"]["share_of_step"] <= 1.0
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
              "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["higher_is_better"] is False and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert "workload" in d["config"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["roofline"]["bound"] in ("hbm", "tensor")
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["gpu_launches"] > 0 and d["parity"]["rel"] <= d["parity"]["tol"]
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def test_tile_size_limit_before_device(tb):
    """Tiles above 2048 rows are refused before any device work (ValueError),
    instead of being compressed on truncated columns."""
    xy = np.random.default_rng(0).random((3000, 2))
    with pytest.raises(ValueError):
        tb.Handle(xy, 2500)
