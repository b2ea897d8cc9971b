"""Summarise the ncu outputs of tools/profile.sh into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py <tag> [--round 01]

Writes profiles/ncu_r<round>_launches.csv (the raw launch list), profiles/ncu_r<round>_summary.json
(per-kernel share of the step, and the full-set metrics of the dominant SpMM launch) and
profiles/traffic.json (DRAM bytes of that launch, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    # tcgen05 evidence (K5): UTCHMMA ops, tensor sub-pipe, TMEM pipe, TMA bytes
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.per_cycle_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "l2__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
]


UNIT_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
UNIT_NS = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}


def launches(tag):
    """Per launch: (kernel, duration ns, dram bytes read+write or None)."""
    path = os.path.join(OUT, tag + "_launches.csv")
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = collections.OrderedDict()
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else 0.0
        u = r.get("Metric Unit", "")
        d = per.setdefault(key, {"t": 0.0, "bytes": 0.0, "has_bytes": False})
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["t"] = v * UNIT_NS.get(u, 1.0)
        elif r["Metric Name"].startswith("dram__bytes"):
            d["bytes"] += v * UNIT_BYTES.get(u, 1.0)
            d["has_bytes"] = True
    rows = [(k[1], d["t"], d["bytes"] if d["has_bytes"] else None) for k, d in per.items()]
    return path, rows


def have_full(tag, suffix):
    return any(os.path.exists(os.path.join(OUT, tag + suffix + e)) for e in (".ncu-rep", "_raw.csv"))


def full(tag, suffix="_full"):
    rep = os.path.join(OUT, tag + suffix + ".ncu-rep")
    raw_csv = os.path.join(OUT, tag + suffix + "_raw.csv")
    if os.path.exists(rep):
        raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    else:                               # exported on the box by tools/profile.sh
        with open(raw_csv) as fh:
            raw = fh.read()
    rows = list(csv.reader([l for l in raw.splitlines() if l.startswith('"')]))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))
    out = {"kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size")}
    for k in FULL_METRICS:
        if k in d:
            out[k] = d[k]
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v.replace(".", "", 1).isdigit()}
    tot = sum(stalls.values()) or 1.0
    out["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    return rep, out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("tag")
    p.add_argument("--round", default="01")
    a = p.parse_args()
    os.makedirs(PROF, exist_ok=True)
    summary = {"tag": a.tag}
    path, rows = launches(a.tag)
    shutil.copy(path, os.path.join(PROF, "ncu_r%s_launches.csv" % a.round))
    by = collections.OrderedDict()
    for name, t, b in rows:
        key = name.split("(")[0].split("<")[0].replace("void ", "").replace("sten::", "").strip()
        e = by.setdefault(key, {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
        e["launches"] += 1
        e["time_ns"] += t
        e["dram_bytes"] += b or 0.0
    total = sum(v["time_ns"] for v in by.values())
    summary["launch_list"] = {k: {"launches": v["launches"], "time_ns_total": round(v["time_ns"], 1),
                                  "share_of_step": round(v["time_ns"] / total, 4),
                                  "dram_bytes_per_launch": round(v["dram_bytes"] / v["launches"], 1)}
                              for k, v in by.items()}
    summary["note"] = ("ncu launch list of `bench.py --profile --no-graph --lanes 1` (cold caches, serialised "
                       "launches): compare shares, not absolute times")
    rep, f = full(a.tag)
    summary["dominant_launch_full_set"] = f
    if have_full(a.tag, "_tc_full"):
        _, ftc = full(a.tag, "_tc_full")
        ftc["note"] = "C3 1024x4096x16384 1:4 g=64 bf16, tcgen05 kernel (K5), first launch"
        summary["tcgen05_launch_full_set"] = ftc
    if have_full(a.tag, "_sp_full"):
        _, fsp = full(a.tag, "_sp_full")
        fsp["note"] = "K1 sparsify of the dominant case (768x3072 2:4 g=4 fp32)"
        summary["sparsify_launch_full_set"] = fsp
    # the exported CSVs of the full captures travel into profiles/ (raw metrics + details page)
    for suffix, name in (("_full", "dominant"), ("_tc_full", "tcgen05"), ("_sp_full", "sparsify")):
        for page in ("raw", "details"):
            src = os.path.join(OUT, "%s%s_%s.csv" % (a.tag, suffix, page))
            if os.path.exists(src):
                shutil.copy(src, os.path.join(PROF, "ncu_r%s_%s_%s.csv" % (a.round, name, page)))
    with open(os.path.join(PROF, "ncu_r%s_summary.json" % a.round), "w") as fh:
        json.dump(summary, fh, indent=1)
    spmm = [v for k, v in summary["launch_list"].items() if k.startswith("spmm")]
    if spmm:
        with open(os.path.join(PROF, "traffic.json"), "w") as fh:
            json.dump({"spmm_dram_bytes_per_launch": max(s["dram_bytes_per_launch"] for s in spmm) and
                       round(sum(s["dram_bytes_per_launch"] * s["launches"] for s in spmm) /
                             sum(s["launches"] for s in spmm), 1),
                       "source": "profiles/ncu_r%s_launches.csv (dram__bytes_read.sum + dram__bytes_write.sum, "
                                 "mean over the step's SpMM launches)" % a.round}, fh, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
