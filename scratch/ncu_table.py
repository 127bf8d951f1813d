# one-line metric summary per ncu report (units normalised): kernel, us, DRAM MB, DRAM % of peak,
# IMMA pipe %, issue-active %
import csv, subprocess, sys
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
      "msecond": 1e3, "nsecond": 1e-3, "%": 1, "": 1}
def row(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    if len(r) < 3:
        return None
    h, u, v = r[0], r[1], r[2]
    def g(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * SC.get(u[i], 1)
    return {"kernel": v[h.index("Kernel Name")].split("(")[0], "us": g("gpu__time_duration.sum"),
            "dram_MB": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) / 1e6,
            "dram_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "imma_pct": g("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"),
            "tensor_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active")}
if __name__ == "__main__":
    for rep in sys.argv[1:]:
        d = row(rep)
        print(rep.split("/")[-1], d and {k: (round(x, 2) if isinstance(x, float) else x) for k, x in d.items()})
