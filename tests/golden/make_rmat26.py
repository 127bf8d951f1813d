"""Generate tests/golden/rmat26_ef16.json ON THE GPU BOX (the reference's own
generator takes ~17 min and ~34 GB at s26, so the graph comes
from the device generator, which is bit-identical to rmat_graph at every
scale the tests pin: tests/test_gpu_parity.py::test_gpu_rmat_bit_identical):

    python tests/golden/make_rmat26.py  [out.json]   (default gpurun_out/rmat26_ef16.json)

Sources of every field:
* the CSR: tcmis_gen_rmat(26, 16, 1) on cuda:0, downloaded; its checksums;
* H2 / luby-perm MIS membership and per-round selected / removed / alive:
  the UNMODIFIED reference (oracle/_ref) run_luby_reference(Permutation) on
  that CSR -- the same MIS and rounds as run_tc_mis(H2), whose
  tiled path would need ~237 GB of tiles here;
* the same membership re-pinned by the reference's own test oracle
  sequential_greedy_mis (proj/tests/support/oracles.cpp:76-92) under the
  reference's h2_degree_aware priorities;
* per-round tiles_evaluated / tiles_skipped at T = 16 (H2, H1) and H3's
  collapsed iteration, and H1's trajectory: the C restatement (oracle/), whose
  tile counters are pinned against the reference's run_tc_mis at every
  BASELINE config that fits (tests/golden/rmat22_ef16.json etc.) -- here it
  must also reproduce the reference's H2 selected / removed / alive exactly,
  which the script asserts.
Run on the GPU box only (reads nothing from /root/reference; oracle/_ref
travels with the snapshot).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2605_29604_b200 as tc  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def rounds5(rr):
    return [[int(r["sel"]), int(r["rem"]), int(r["alive"]), int(r["tiles_eval"]),
             int(r["tiles_skip"])] for r in rr]


def main():
    scale = int(os.environ.get("TCMIS_GOLDEN_SCALE", "26"))  # smaller: a dry run of the script
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out",
                                                                   f"rmat{scale}_ef16.json")
    t0 = time.time()
    if os.environ.get("TCMIS_GOLDEN_CPU"):  # dry run without a GPU: the oracle's generator
        g = O.gen("rmat", scale, 16, 1)
    else:
        ctx = tc.Context(0)
        dg = tc.DeviceGraph.rmat(scale, 16, 1, ctx)
        h = dg.download()
        dg.close()
        g = O.Graph(h.n, h.offsets, h.neighbors)
    deg = np.diff(g.off)
    log(f"generated + downloaded s{scale}: n={g.n} nnz={g.nbr.size} ({time.time() - t0:.0f}s)")
    out = {"name": f"rmat{scale}_ef16",
           "source": "tests/golden/make_rmat26.py on a B200 box: CSR from the device generator "
                     "(bit-identical to rmat_graph), H2/luby-perm membership and rounds from the "
                     "unmodified reference's run_luby_reference(Permutation), re-pinned by the "
                     "reference's sequential_greedy_mis; tile counters, H1 and H3 from the C "
                     "restatement (oracle/), which reproduces the reference's H2 rounds here",
           "spec": {"kind": "rmat", "scale": scale, "ef": 16, "seed": 1},
           "n": g.n, "m": g.num_edges, "off_checksum": O.checksum(g.off),
           "nbr_checksum": O.checksum(g.nbr), "max_degree": int(deg.max()), "tile_dim": 16}
    R = O.ref()
    rg = O.RefGraph.from_csr(g)
    cores = os.cpu_count() or 1
    t1 = time.time()
    member, rr, ms = O.ref_run_luby(rg, 1, False, 20, cores)
    log(f"reference run_luby_reference(Permutation): {len(rr)} rounds, |MIS| "
        f"{int(member.sum())}, {ms:.0f} ms ({time.time() - t1:.0f}s)")
    ref_member = member.astype(np.uint8)
    ref_rounds = [[int(r["sel"]), int(r["rem"]), int(r["alive"])] for r in rr]
    # the reference's test oracle: greedy MIS in (p, id) order
    p = np.zeros(g.n, np.uint32)
    assert R.ref_h2_degree_aware(rg.h, 1, 20, p) == 0
    greedy = np.zeros(g.n, np.uint8)
    R.ref_sequential_greedy(rg.h, p, greedy)
    assert np.array_equal(greedy, ref_member), "sequential_greedy_mis disagrees"
    del rg
    # tile counters (T = 16) and the other heuristics from the restatement
    t2 = time.time()
    rt = O.tile_row_counts(g, 16)
    out["tile_count"] = int(rt.sum())
    log(f"oracle T=16 tiles per block column: {out['tile_count']} ({time.time() - t2:.0f}s)")
    results = {}
    po = O.priorities(g, "h2", 1, 20)
    assert np.array_equal(po, p), "oracle h2 priorities differ from the reference's"
    t3 = time.time()
    s2 = O.luby_rounds(g, po, T=16, col_counts=rt)
    log(f"oracle h2 rounds ({time.time() - t3:.0f}s)")
    assert np.array_equal((s2.state == 1).astype(np.uint8), ref_member)
    r2 = rounds5(s2.rounds)
    assert [r[:3] for r in r2] == ref_rounds, (r2, ref_rounds)
    member_ck = O.checksum(ref_member)
    mis = int(ref_member.sum())
    results["h2/seed1"] = {"rounds": r2, "mis_size": mis, "member_checksum": member_ck,
                           "ref_wall_ms": ms,
                           "terms": [[int(r["alive_start"]), int(r["nnz_alive"]),
                                      int(r["noncand"]), int(r["nnz_noncand"]),
                                      int(r["nnz_cand"])] for r in s2.rounds]}
    results["luby-perm/seed1"] = {"rounds": [r + [0, 0] for r in ref_rounds], "mis_size": mis,
                                  "member_checksum": member_ck, "ref_wall_ms": ms}
    seg = np.zeros(rt.size, bool)
    seg[np.flatnonzero(ref_member) // 16] = True
    ev = int(rt[seg].sum())
    results["h3/seed1"] = {"rounds": [[mis, g.n - mis, 0, ev, out["tile_count"] - ev]],
                           "mis_size": mis, "member_checksum": member_ck}
    t4 = time.time()
    s1 = O.luby_rounds(g, O.priorities(g, "h1", 1), T=16, col_counts=rt)
    m1 = (s1.state == 1).astype(np.uint8)
    log(f"oracle h1 rounds: {s1.n_rounds} ({time.time() - t4:.0f}s)")
    results["h1/seed1"] = {"rounds": rounds5(s1.rounds), "mis_size": int(m1.sum()),
                           "member_checksum": O.checksum(m1)}
    out["results"] = results
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    log(f"wrote {out_path} ({time.time() - t0:.0f}s)")


if __name__ == "__main__":
    main()
