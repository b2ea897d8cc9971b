"""Summarise tools/profile_r02.sh outputs (gpurun_out/r02_*) into profiles/ (runs here, no GPU):
profiles/ncu_r02_launches.csv (raw launch list of the bench step), profiles/ncu_r02_summary.json
(per-kernel share of the step + the selected full-set metrics of each captured kernel) and
profiles/traffic_r02.json (DRAM bytes of the dominant launch per config, read by bench.py)."""
import collections
import csv
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = os.environ.get("TAG", "r02")        # r02b: the second profiling pass of round 2 (tools/profile_r02b.sh)
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
UNIT = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l2__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def csv_rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    return list(csv.reader(lines))


def launch_list():
    rows = csv_rows(os.path.join(OUT, TAG + "_launches.csv"))
    h = rows[0]
    I, K, N, U, V = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per, names = collections.defaultdict(dict), {}
    for r in rows[1:]:
        per[r[I]][r[N]] = float(r[V].replace(",", "")) * UNIT.get(r[U], 1.0)
        names[r[I]] = r[K]
    tot, cnt, dram = collections.Counter(), collections.Counter(), collections.Counter()
    for i, d in per.items():
        k = names[i].split("(")[0].replace("void ", "")
        tot[k] += d.get("gpu__time_duration.sum", 0.0)
        dram[k] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        cnt[k] += 1
    T = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "time_us": round(v / 1e3, 2), "share": round(v / T, 4),
             "dram_bytes_per_launch": round(dram[k] / cnt[k])} for k, v in tot.most_common()]


def full(name):
    path = os.path.join(OUT, "%s_%s_raw.csv" % (TAG, name))
    if not os.path.exists(path):
        return None
    rows = csv_rows(path)
    h, u = rows[0], rows[1]
    out = {}
    for row in rows[2:3]:
        d = dict(zip(h, row))
        du = dict(zip(h, u))
        out["kernel"] = d.get("Kernel Name", "")[:120]
        for k in KEYS:
            if k in d:
                out[k] = [d[k], du.get(k, "")]
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v.replace(",", "").replace(".", "", 1).isdigit()}
        s = sum(st.values()) or 1.0
        out["stalls_pct"] = {k: round(100 * v / s, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]}
    return out


def main():
    ll = launch_list()
    shutil.copy(os.path.join(OUT, TAG + "_launches.csv"), os.path.join(PROF, "ncu_%s_launches.csv" % TAG))
    summ = {"_what": "round 2, one B200: ncu launch list of `bench.py --profile --steps 2 --warmup 1 --no-graph` "
                     "(the grouped C2 step; serialised, cold: compare shares) and --set full captures "
                     "(tools/profile_%s.sh)" % TAG, "launch_list": ll}
    for name in ("grouped", "gsparsify", "sp24", "sddmm", "nmgx"):
        summ[name] = full(name)
    with open(os.path.join(PROF, "ncu_%s_summary.json" % TAG), "w") as f:
        json.dump(summ, f, indent=1)
    g = summ.get("grouped")
    if g and "dram__bytes_read.sum" in g:
        b = sum(float(g[k][0].replace(",", "")) * UNIT.get(g[k][1], 1.0)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        with open(os.path.join(PROF, "traffic_r02.json"), "w") as f:
            json.dump({"_what": "dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the dominant kernel, "
                                "ncu --set full (tools/profile_r02.sh)",
                       "c1_f32_grouped": {"kernel": g["kernel"], "dram_bytes_per_launch": round(b)}}, f, indent=1)
    print(json.dumps(ll[:6], indent=1))


if __name__ == "__main__":
    main()
