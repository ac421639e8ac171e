"""Summarise ncu outputs from gpurun_out/ into profiles/ (launch shares + full-set metrics).

    python scripts/ncu_summary.py TAG            # every gpurun_out/prof_*.raw.csv (scripts/prof_final.sh)
    python scripts/ncu_summary.py TAG REP.ncu-rep  # one report

Per capture: duration, DRAM bytes read/written (the roofline "traffic"), DRAM
throughput, SM / L1 / L2 throughput, tensor-pipe instructions, registers, grid,
warp stall mix.  The launch list gives each kernel family's share of the GPU
time of `bench.py --steps 2 --warmup 1` (ncu --metrics gpu__time_duration.sum).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.sum", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__m_l1tex2xbar_write_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "smsp__cycles_active.avg", "gpc__cycles_elapsed.max",
        # tensor pipe (tcgen05 UTCHMMA = the TF32 / F16 MMAs) and tensor memory
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


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


def _rows(raw_text):
    r = list(csv.reader(io.StringIO(raw_text)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        if len(row) != len(hdr):
            continue
        d = {"kernel": row[hdr.index("Kernel Name")][:140]}
        for w in WANT:
            # raw-page headers may carry a section prefix ("TPC.TriageCompute.<metric>")
            idx = [k for k, h in enumerate(hdr) if h == w or h.endswith("." + w)]
            if idx:
                d[w] = f"{row[idx[0]]} {units[idx[0]]}".strip()
        try:
            rd = float(row[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(row[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            d["dram_traffic_bytes"] = int(rd * scale[units[hdr.index("dram__bytes_read.sum")]] +
                                          wr * scale[units[hdr.index("dram__bytes_write.sum")]])
        except (ValueError, KeyError):
            pass
        res.append(d)
    return res


def full(path):
    if path.endswith(".csv"):
        return _rows(open(path).read())
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return _rows(raw)


if __name__ == "__main__":
    tag = sys.argv[1]
    out = {}
    if os.path.exists("gpurun_out/launches.csv"):
        out["launch_list"] = launches("gpurun_out/launches.csv")
    srcs = sys.argv[2:] or sorted(glob.glob("gpurun_out/prof_*.raw.csv"))
    out["captures"] = {}
    for s in srcs:
        name = os.path.basename(s).replace(".raw.csv", "").replace(".ncu-rep", "")
        try:
            out["captures"][name] = full(s)
        except Exception as e:  # noqa: BLE001
            out["captures"][name] = {"error": str(e)}
    json.dump(out, open(f"profiles/{tag}.json", "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])
