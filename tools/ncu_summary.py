#!/usr/bin/env python3
"""Summarise ncu reports (run here, on the CPU box) into profiles/ncu_summary.json (merged: kernels
captured in these reports replace their earlier entries).

    python tools/ncu_summary.py gpurun_out/prof_r1.ncu-rep [more.ncu-rep ...] [--launches launches.csv]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed_pipe_fma.sum": "inst_pipe_fma",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": "thread_ffma",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": "thread_ffma",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_ld_bank_conflicts",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "sm__pipe_fma_cycles_active.sum.pct_of_peak_sustained_active": "fma_pipe_active_pct",
    "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active": "fma_pipe_inst_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_smem_operand_active_pct",
}


DIRECT = ("k_res_s", "k_grad_s", "k_tc_dense", "k_absmax2", "k_residual_gather", "k_scatter_real", "k_conv_residual", "k_conv_rows", "k_conv_dense", "k_ista_update", "k_residual_reduce", "k_admm_beta",
          "k_admm_x", "k_admm_duals", "k_metrics_final")
FFT = ("k_fft_pass<16, -1>", "k_fft_pass<16, 1>", "k_fft_pass<8, -1>", "k_fft_pass<8, 1>", "k_fft_pass<4, -1>",
       "k_fft_pass<4, 1>", "k_fft_pass<2, -1>", "k_fft_pass<2, 1>", "k_real_to_complex", "k_spec_mul",
       "k_extract_real", "k_gather_real", "k_zero_c", "k_scatter_rows", "k_rows_r2c", "k_mid", "k_cols_fwd",
       "k_cols_inv", "k_rows")


def short(name):
    for k in DIRECT + FFT + ("k_ffma_peak",):
        if k in name:
            return k
    return name.split("(")[0][-40:]


def group(k):
    # k_residual_reduce / k_ista_update are shared by both engines; attribute them to the direct step
    return "direct_engine" if k in DIRECT else "fft_engine" if k in FFT else "other"


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": short(d.get("Kernel Name", "")), "report": os.path.basename(rep)}
        for k, v in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    e[v] = float(d[k].replace(",", "")) * scale.get(units.get(k, ""), 1.0)
                except ValueError:
                    pass
        if "dram_read_bytes" in e:
            e["dram_bytes_per_launch"] = e["dram_read_bytes"] + e.get("dram_write_bytes", 0.0)
            if e.get("duration_ns"):
                e["dram_gbs"] = e["dram_bytes_per_launch"] / e["duration_ns"]  # bytes/ns = GB/s
        stalls = {}
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(d[k])
                except ValueError:
                    pass
        e["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        res.append(e)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = {}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = {}
    for k, v in agg.items():
        tot[group(k)] = tot.get(group(k), 0.0) + v[1]
    return {k: {"launches": v[0], "total_ns": v[1], "mean_ns": v[1] / v[0], "group": group(k),
                "share_of_group": v[1] / tot[group(k)]}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    args = sys.argv[1:]
    lp = None
    if "--launches" in args:
        i = args.index("--launches")
        lp = args[i + 1]
        del args[i:i + 2]
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
    try:  # merge: kernels captured here replace their earlier entries, the others stay
        summary = json.load(open(dst))
    except (OSError, ValueError):
        summary = {}
    fresh = set()
    for rep in args:
        for e in load(rep):
            if e["kernel"] not in fresh:  # first capture of each kernel in this run
                summary[e["kernel"]] = e
                fresh.add(e["kernel"])
    if lp:
        summary["launch_list"] = launches(lp)
        summary["launch_list_source"] = os.path.basename(lp)
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
