"""Summarise ncu outputs from gpurun_out/ into profiles/ (launch shares + full-set metrics)."""
import csv, io, json, subprocess, sys
from collections import defaultdict

def launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "avg_us": round(sum(v) / len(v) / 1e3, 3),
                    "share": round(sum(v) / tot, 4)})
    return out

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.sum", "launch__grid_size", "launch__block_size",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]

def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")][:120]}
        for w in WANT:
            if w in hdr:
                d[w] = f"{row[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        res.append(d)
    return res

if __name__ == "__main__":
    tag = sys.argv[1]
    out = {"launch_list": launches("gpurun_out/launches.csv")}
    try:
        out["full_set"] = full(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/prof_full.ncu-rep")
    except Exception as e:
        out["full_set_error"] = str(e)
    json.dump(out, open(f"profiles/{tag}.json", "w"), indent=1)
    print(json.dumps(out, indent=1)[:4000])
