"""Generate tests/golden/*.json from the REFERENCE compiled from its own
sources (oracle/_ref/libtcmis_ref.so) -- run here, in the build container,
where /root/reference exists:

    python tests/golden/make_golden.py [small|large|all]

Graphs: ER and R-MAT come from the reference generators themselves
(gnp_graph_avg_degree / rmat_graph); the grid and the RGG have no reference
generator and come from the oracle's definitions (oracle/tcmis_oracle.c,
DESIGN.md "Synthetic inputs").  Every MIS, round trajectory and tile counter
comes from the reference engine (run_tc_mis over tile_graph, run_luby_reference).
The oracle contributes only the per-round byte-model terms (alive_start,
nnz_alive, noncand, nnz_noncand), checked against the reference's round stats.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R = O.ref()


def graph_for(spec):
    kind = spec["kind"]
    if kind == "rmat":
        rg = O.RefGraph(R.ref_gen_rmat(spec["scale"], spec["ef"], spec["seed"]))
        return rg, rg.to_csr()
    if kind == "gnp":
        rg = O.RefGraph(R.ref_gen_gnp_avg(spec["n"], spec["d"], spec["seed"]))
        return rg, rg.to_csr()
    if kind == "grid":
        g = O.gen("grid", spec["side"])
    elif kind == "rgg":
        g = O.gen("rgg", spec["n"], spec["d"], spec["seed"])
    elif kind == "petersen":
        g = O.gen("petersen")
    else:
        raise ValueError(kind)
    return O.RefGraph.from_csr(g), g


def rounds_of(rr):
    return [[int(r["sel"]), int(r["rem"]), int(r["alive"]), int(r["tiles_eval"]),
             int(r["tiles_skip"])] for r in rr]


def make(name, spec, heuristics=("h2", "h3", "h1", "luby-perm"), seeds=(1,), T=16):
    t0 = time.time()
    rg, g = graph_for(spec)
    out = {"name": name, "spec": spec, "n": g.n, "m": g.num_edges,
           "off_checksum": O.checksum(g.off), "nbr_checksum": O.checksum(g.nbr),
           "max_degree": int(np.diff(g.off).max()) if g.n else 0, "tile_dim": T}
    ms = O.C.c_double(0)
    tiled = R.ref_tile_graph(rg.h, T, O.C.byref(ms))
    out["tile_count"] = int(R.ref_tiled_count(tiled))
    out["tile_graph_ms"] = ms.value
    res = {}
    for seed in seeds:
        for h in heuristics:
            member = np.zeros(max(g.n, 1), np.uint8)
            cnt = O.C.c_int64(0)
            rounds = (O.RefRound * 4096)()
            nr = O.C.c_int(0)
            wall = O.C.c_double(0)
            if h == "luby-perm":
                rc = R.ref_run_luby(rg.h, seed, 0, 20, 0, member, O.C.byref(cnt), rounds, 4096,
                                    O.C.byref(nr), O.C.byref(wall))
            else:
                rc = R.ref_run_tc_mis_tiled(rg.h, tiled, O.HEURISTICS[h], seed, T, 0, 20, member,
                                            O.C.byref(cnt), rounds, 4096, O.C.byref(nr),
                                            O.C.byref(wall))
            assert rc == 0, O.ref().ref_last_error()
            rr = [{f: getattr(rounds[i], f) for f, _ in O.RefRound._fields_}
                  for i in range(nr.value)]
            entry = {"rounds": rounds_of(rr), "mis_size": int(cnt.value),
                     "member_checksum": O.checksum(member[:g.n]), "ref_wall_ms": wall.value}
            if h in ("h2", "h1"):  # byte-model terms from the oracle, pinned to the ref stats
                p = O.priorities(g, h, seed)
                s = O.luby_rounds(g, p, T=T)
                assert [[r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"]]
                        for r in s.rounds] == entry["rounds"], (name, h, "oracle != reference")
                assert O.checksum((s.state == 1).astype(np.uint8)) == entry["member_checksum"]
                entry["terms"] = [[r["alive_start"], r["nnz_alive"], r["noncand"],
                                   r["nnz_noncand"], r["nnz_cand"]] for r in s.rounds]
            res[f"{h}/seed{seed}"] = entry
    R.ref_tiled_free(tiled)
    out["results"] = res
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: n={g.n} m={g.num_edges} tiles={out['tile_count']} "
          f"({time.time() - t0:.1f}s)", flush=True)


SMALL = {
    "petersen": {"kind": "petersen"},
    "gnp1000_d8_s7": {"kind": "gnp", "n": 1000, "d": 8.0, "seed": 7},
    "rmat10_ef16_s3": {"kind": "rmat", "scale": 10, "ef": 16, "seed": 3},
    "rmat14_ef16_s1": {"kind": "rmat", "scale": 14, "ef": 16, "seed": 1},
    "grid64": {"kind": "grid", "side": 64},
    "rgg20k_d3_s1": {"kind": "rgg", "n": 20000, "d": 3.0, "seed": 1},
}
LARGE = {
    "er_n100k_d16": {"kind": "gnp", "n": 100000, "d": 16.0, "seed": 1},
    "grid4096": {"kind": "grid", "side": 4096},
    "rmat22_ef16": {"kind": "rmat", "scale": 22, "ef": 16, "seed": 1},
    "rgg24m_d3": {"kind": "rgg", "n": 24000000, "d": 3.0, "seed": 1},
}

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which in ("small", "all"):
        for k, v in SMALL.items():
            make(k, v, seeds=(1, 2, 3))
    if which in ("large", "all"):
        for k, v in LARGE.items():
            if len(sys.argv) > 2 and k not in sys.argv[2:]:
                continue
            make(k, v, heuristics=("h2", "h3", "h1"))
