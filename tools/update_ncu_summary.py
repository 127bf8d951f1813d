# profiles/ncu_summary.json from ncu launch lists (gpu__time_duration + dram
# bytes) of tools/ncu_target.py: per config, the round-1 launch of every
# kernel in the SECOND (warm) solve.  usage: update_ncu_summary.py CFG CSV [CFG CSV ...]
import csv, json, os, re, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
try:
    summ = json.load(open(out_path))
except Exception:
    summ = {}
summ["_doc"] = ("per config: ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                "dram__bytes_write.sum --clock-control none) of tools/ncu_target.py; the round-1 "
                "launch of each kernel in the second (warm) host-loop solve; dram_bytes = read + write "
                "per launch (cold-cache, serialised by ncu)")
args = sys.argv[1:]
for cfg, path in zip(args[::2], args[1::2]):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = launches.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        k[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    seq = [launches[i] for i in sorted(launches)]
    # a solve starts with k_priorities, or on the degree order k_init_ctrl +
    # k_prio_settle (the fused init)
    starts = [i for i, k in enumerate(seq)
              if "k_priorities" in k["name"] or "k_init_ctrl" in k["name"]]
    if not starts:
        continue
    solve = seq[starts[-1]:]
    entry = {"source": os.path.basename(path)}
    for k in solve:
        m = re.search(r"(k_[a-z0-9_]+)", k["name"])
        short = m.group(1) if m else k["name"][:40]
        if short in entry:
            continue  # round 1 = first launch of the solve
        tb = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        entry[short] = {"dram_bytes": int(tb), "duration_us": k.get("gpu__time_duration.sum", 0) / 1e3}
    summ[cfg] = entry
json.dump(summ, open(out_path, "w"), indent=1)
print({c: sorted(v) for c, v in summ.items() if isinstance(v, dict)})
