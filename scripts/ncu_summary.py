"""Summarise ncu captures into profiles/ (run here, without a GPU).

    python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [--dets N]
    python scripts/ncu_summary.py launches <launches.csv> <out.json>

full:     one `ncu --set full` capture of scan_kernel -> key metrics (duration, DRAM bytes,
          FP64 pipe / issue utilisation, occupancy, stall reasons, executed FP64 ops).
          --dets: algorithmic determinants of the captured launch (masw_last_work), to
          express per-det instruction counts and the algorithmic FLOP rate.
launches: `ncu --metrics gpu__time_duration.sum` launch list -> per-kernel time share.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res


_UNITS = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
          "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
          "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def num(d, k, si=False):
    """Metric value; with si=True converted to seconds / hertz / bytes from its unit."""
    v, u = d.get(k, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * _UNITS.get(u, 1.0) if si else x


def full(rep, out, dets=None):
    launches = raw_metrics(rep)
    summary = []
    for d in launches:
        dur_s = num(d, "gpu__time_duration.sum", si=True)
        rd = num(d, "dram__bytes_read.sum", si=True) or 0.0
        wr = num(d, "dram__bytes_write.sum", si=True) or 0.0
        dfma = num(d, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum")
        dadd = num(d, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum")
        dmul = num(d, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum")
        rate_keys = {
            "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
            "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
            "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"}
        rates = {k: num(d, v) for k, v in rate_keys.items()}
        s = {
            "kernel": d.get("Kernel Name", ("", ""))[0],
            "duration_ms": dur_s * 1e3 if dur_s else None,
            "sm_mhz": (num(d, "sm__cycles_elapsed.avg.per_second", si=True) or 0) / 1e6 or None,
            "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes": rd + wr,
            "fp64_pipe_pct_active": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_inst_pct_active": num(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            # issue utilisation = cycles in which the SMSP issued an instruction; NOT
            # sm__instruction_throughput (a max-over-pipes roll-up, = the busiest pipe)
            "issue_slots_busy_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "instruction_throughput_pct": num(d, "sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": num(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": num(d, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "xu_pipe_pct": num(d, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "ipc": num(d, "sm__inst_executed.avg.per_cycle_active"),
            "warp_inst_executed": num(d, "smsp__inst_executed.sum"),
            "registers_per_thread": num(d, "launch__registers_per_thread"),
            "achieved_occupancy_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "theoretical_occupancy_pct": num(d, "sm__maximum_warps_per_active_cycle_pct"),
            "fp64_thread_ops_per_cycle": rates,
        }
        stalls = {}
        for k, (v, u) in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        s["stall_per_issue_top"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
        if all(v is not None for v in rates.values()) and s["sm_mhz"]:
            flops_per_cycle = 2 * rates["dfma"] + rates["dadd"] + rates["dmul"]
            s["hw_fp64_tflops"] = flops_per_cycle * s["sm_mhz"] * 1e6 / 1e12
            s["hw_fp64_frac_of_derived_peak"] = flops_per_cycle / (148 * 64 * 2)
        if dets and s["warp_inst_executed"]:
            s["algorithmic_dets"] = dets
            if s["duration_ms"]:
                s["algorithmic_dets_per_s"] = dets / (s["duration_ms"] / 1e3)
            s["thread_inst_per_det"] = s["warp_inst_executed"] * 32 / dets
            s["dram_bytes_per_det"] = s["dram_bytes"] / dets
        summary.append(s)
    json.dump(summary if len(summary) > 1 else summary[0], open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


def launches(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
                 "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1e-6)
        ms = v * scale
        name = r["Kernel Name"].split("(")[0]
        per[name][0] += 1
        per[name][1] += ms
        total += ms
    res = {"total_ms": total, "launches": sum(v[0] for v in per.values()),
           "kernels": {k: {"launches": v[0], "ms": v[1], "share": v[1] / total if total else None}
                       for k, v in sorted(per.items(), key=lambda x: -x[1][1])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        dets = None
        if "--dets" in sys.argv:
            dets = float(sys.argv[sys.argv.index("--dets") + 1])
        full(sys.argv[2], sys.argv[3], dets)
    else:
        launches(sys.argv[2], sys.argv[3])
