"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
the engine refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2605_29604_b200 as tc
from conftest import ROOT


def declared_symbols(header: str):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcmis_[a-z0-9_]+)\s*\(", src)))


def exported(lib: str):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_exports_every_declared_symbol():
    assert os.path.exists(tc.library_path()), "build the library first"
    syms = declared_symbols("tcmis_b200.h")
    assert len(syms) >= 30
    have = exported(tc.library_path())
    missing = [s for s in syms if s not in have]
    assert not missing, missing
    lib = tc.load()
    for s in syms:
        assert hasattr(lib, s)


def test_only_the_c_abi_is_exported():
    have = exported(tc.library_path())
    ours = {s for s in have if s.startswith("tcmis_")}
    # kernels and helpers stay hidden (-fvisibility=hidden)
    assert not any("tcmis_b200" in s for s in have - ours if s.startswith("_Z"))


def test_cxx_dropin_library_exports_engine_api():
    lib = os.path.join(ROOT, "paper_2605_29604_b200", "libtcmis.so")
    if not os.path.exists(lib):
        pytest.skip("libtcmis.so not built")
    names = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True,
                           check=True).stdout
    for sym in ("tcmis::b200::run_mis(", "tcmis::b200::run_tc_mis(", "tcmis::b200::tile_graph(",
                "tcmis::b200::h2_degree_aware(", "tcmis::b200::h1_random(",
                "tcmis::b200::compute_max_np(",
                "tcmis::b200::tiled_spmv(", "tcmis::b200::phase3_update(",
                "tcmis::b200::run_h3_resolution(", "tcmis::b200::write_tiled(",
                "tcmis::b200::read_tiled(", "tcmis::b200::tile_stats(",
                "tcmis::b200::check_independence(", "tcmis::b200::check_maximality(",
                "tcmis::b200::csv_header[abi:cxx11](", "tcmis::b200::csv_row("):
        assert sym in names, sym


def test_config_defaults_match_engine_hpp():
    c = tc._Config()
    tc.load().tcmis_config_init(ctypes.byref(c))
    assert (c.heuristic, c.tile_dim, c.seed, c.scale_bits, c.workers) == (2, 16, 1, 20, 0)
    assert tc.EngineConfig().heuristic == tc.Heuristic.H3


def test_heuristic_names():
    for h in tc.Heuristic:
        assert tc.heuristic_from_name(tc.heuristic_name(h)) == h
    with pytest.raises(ValueError):
        tc.heuristic_from_name("h4")


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tc.CudaError):
        tc.Context(0)


def test_rgg_radius_definition():
    import math
    n = 24_000_000
    assert tc.rgg_radius(n, 3.0) == math.floor(math.sqrt(3.0 / (math.pi * n)) * 2**32)
    import oracle as O
    assert tc.rgg_radius(n, 3.0) == O.lib().orc_rgg_radius(n, 3.0)
