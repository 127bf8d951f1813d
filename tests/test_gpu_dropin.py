"""GPU: a C++ program written against the reference's public headers
(tests/cpp/dropin_main.cpp), compiled against include/tcmis/*.hpp and linked
with libtcmis.so, gives the reference's results (checked with the oracle)."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import ROOT

pytestmark = pytest.mark.gpu

PKG = os.path.join(ROOT, "paper_2605_29604_b200")


def fnv_ids(ids):
    h = 0xcbf29ce484222325
    for x in ids.tolist():
        h ^= x & 0xFFFFFFFF
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.fixture(scope="module")
def dropin(tmp_path_factory):
    d = tmp_path_factory.mktemp("dropin")
    exe = str(d / "dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp"), "-L", PKG, "-ltcmis",
                    "-ltcmis_b200", f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe, d


@pytest.mark.parametrize("kind,args", [("rmat", (12, 16, 2)), ("gnp_avg", (3000, 10.0, 5)),
                                       ("grid", (30,))])
@pytest.mark.parametrize("device_edges", [False, True])
def test_cpp_dropin_matches_reference(dropin, kind, args, device_edges, monkeypatch):
    """device_edges: the C++ graph_from_edges (and so the tiled round trip
    and the edge-range error) through the device normaliser at any size."""
    if device_edges:
        monkeypatch.setenv("TCMIS_FROM_EDGES_DEVICE_MIN", "1")
    exe, d = dropin
    g = O.gen(kind, *args)
    path = str(d / f"{kind}.bin")
    with open(path, "wb") as f:
        f.write(np.int32(g.n).tobytes())
        f.write(np.int64(g.nbr.size).tobytes())
        f.write(g.off.astype(np.int64).tobytes())
        f.write(g.nbr.astype(np.int32).tobytes())
    out = subprocess.run([exe, path], capture_output=True, text=True, check=True).stdout
    lines = [json.loads(x) for x in out.strip().splitlines()]
    runs = [x for x in lines if "heuristic" in x]
    assert len(runs) == 10
    for r in runs:
        exp = O.solve(g, r["heuristic"], r["seed"], tile_dim=16)
        assert r["size"] == exp.mis.size
        assert r["mis_fnv"] == fnv_ids(exp.mis)
        assert r["rounds"] == [[x["sel"], x["rem"], x["alive"], x["tiles_eval"], x["tiles_skip"]]
                               for x in exp.rounds]
        want_obs = {"h1": exp.n_rounds, "h2": exp.n_rounds, "h3": 1, "luby-fresh": 0,
                    "luby-perm": 0}[r["heuristic"]]
        assert r["observed"] == want_obs
    tio = [x for x in lines if "tiled_io" in x][0]
    assert (tio["tiled_io"], tio["roundtrip"]) == (1, 1)
    assert tio["nonzeros"] == g.nbr.size
    assert tio["csr_est"] == 8 * (g.n + 1) + 4 * g.nbr.size
    assert [x for x in lines if "bad_magic" in x][0]["bad_magic"] == "yes"
    if O.ref_available():  # byte-identical to the reference's own cache file
        ref_path = path + ".ref.t16"
        O.ref_write_tiled(O.RefGraph.from_csr(g), 16, ref_path)
        with open(path + ".t16", "rb") as a, open(ref_path, "rb") as b:
            assert a.read() == b.read()
    val = [x for x in lines if "valid_ind" in x][0]
    exp2 = O.solve(g, "h2", 1, tile_dim=16)
    mis2 = np.flatnonzero(exp2.state == 1)
    assert (val["valid_ind"], val["valid_max"]) == (1, 1)
    want = O.check_maximality(g, mis2[1:])
    assert (bool(val["minus_first_max"]), val["addable"]) == (want[0], -1 if want[1] is None else want[1])
    t8 = [x for x in lines if "tiles8" in x][0]
    assert t8["tiles8"] == int(O.tile_row_counts(g, 8).sum())
    e8 = O.solve(g, "h2", 1, tile_dim=8)
    assert t8["t8_rounds"] == e8.n_rounds and t8["t8_eval1"] == e8.rounds[0]["tiles_eval"]
    csv = [x for x in lines if "csv_row" in x][0]
    assert csv["csv_header"].split(",") == [
        "graph", "n", "m", "heuristic", "seed", "mis_size", "iterations", "total_ms",
        "phase1_ms", "phase2_ms", "phase3_ms", "tiles_evaluated", "tiles_skipped"]
    row = csv["csv_row"].split(",")
    assert row[:7] == ["g", str(g.n), str(g.num_edges), "h2", "1", str(int(mis2.size)),
                       str(exp2.n_rounds)]
    assert all(float(x) >= 0 for x in row[7:11])
    assert row[11:] == [str(sum(x["tiles_eval"] for x in exp2.rounds)),
                        str(sum(x["tiles_skip"] for x in exp2.rounds))]
    assert csv["csv_bad_name"] == "yes"
    errs = [x for x in lines if "bad_tile" in x][0]
    assert all(v == "yes" for v in errs.values()), errs
