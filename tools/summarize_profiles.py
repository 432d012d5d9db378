#!/usr/bin/env python
"""Turns the raw ncu outputs in gpurun_out/ into the committed summaries under profiles/:

  profiles/r01_launches_<workload>.csv / .md   per-kernel device time and share of a CG iteration
  profiles/r01_ncu_<kernel>_<workload>.txt     key metrics of one `ncu --set full` capture
  profiles/traffic.json                        dram bytes per launch (bench.py's roofline.traffic)

Usage: python tools/summarize_profiles.py   (no GPU needed; reads .ncu-rep with `ncu -i`)
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launch_list(name, workload):
    src = os.path.join(OUT, name)
    if not os.path.exists(src):
        return
    shutil.copy(src, os.path.join(PROF, name))
    with open(src) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    rows = []
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        kernel = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1]
        value = float(r["Metric Value"].replace(",", ""))
        rows.append((kernel, r["Grid Size"] + " x " + r["Block Size"], value / 1000.0 if r["Metric Unit"].startswith("n") else value))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for kernel, grid, us in rows:
        agg[(kernel, grid)][0] += 1
        agg[(kernel, grid)][1] += us
    total = sum(v[1] for v in agg.values())
    by_kernel = collections.defaultdict(float)
    for (kernel, _grid), v in agg.items():
        by_kernel[kernel] += v[1]
    iterations = sum(1 for kernel, _g, _us in rows if kernel.startswith("k_cg_record"))
    out = [f"# ncu launch list — {workload} ({len(rows)} launches captured from the steady state of a solve, {iterations} CG iterations)",
           "", "`ncu --metrics gpu__time_duration.sum --clock-control none` on `bench.py`; per-launch times are cold-cache and",
           "serialised (ncu flushes caches and drops the programmatic overlap), so read the SHARES, not the absolutes.", "",
           "| kernel | grid x block | launches | total µs | avg µs | share |", "|---|---|---|---|---|---|"]
    for (kernel, grid), v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {kernel} | {grid} | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {v[1] / total * 100:.1f} % |")
    out += ["", "| kernel (all grids) | share |", "|---|---|"]
    for kernel, us in sorted(by_kernel.items(), key=lambda kv: -kv[1]):
        out.append(f"| {kernel} | {us / total * 100:.1f} % |")
    with open(os.path.join(PROF, name.replace(".csv", ".md")), "w") as fh:
        fh.write("\n".join(out) + "\n")


WANT = ["smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.max",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "idc__request_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tensor.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def live_list(name, workload):
    """per-kernel duration and DRAM bytes of one eager, steady-state CG iteration pair (tools/ncu_target.py --what
    iteration --count 2) with LIVE caches (--cache-control none): the achieved-HBM table of DESIGN.md §4"""
    src = os.path.join(OUT, name)
    if not os.path.exists(src):
        return
    shutil.copy(src, os.path.join(PROF, name))
    with open(src) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    per = collections.OrderedDict()
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in csv.DictReader(lines):
        d = per.setdefault(r["ID"], {"k": re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1], "grid": r["Grid Size"], "block": r["Block Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v / 1000.0 if r["Metric Unit"].startswith("n") else v
        else:
            d[r["Metric Name"]] = v * scale[r["Metric Unit"]]
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault((d["k"], d["grid"], d["block"]), [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["us"]
        a[2] += d.get("dram__bytes_read.sum", 0.0)
        a[3] += d.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    out = [f"# per-kernel time and DRAM traffic, live caches — {workload} ({len(per)} launches: two eager CG iterations plus the solve's prologue)",
           "", "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none`",
           "on `tools/ncu_target.py --what iteration --count 2` (graphs off so that every kernel is its own row). Launches are",
           "serialised by ncu (no programmatic overlap), caches are NOT flushed between them: the DRAM bytes are what the kernel",
           "moves in the running solve. GB/s = (read + write) / duration against the measured 6 551 GB/s.", "",
           "| kernel | grid | block | launches | avg µs | share | DRAM read MB | DRAM write MB | GB/s | frac of 6 551 |", "|---|---|---|---|---|---|---|---|---|---|"]
    for (k, grid, block), a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = (a[2] + a[3]) / a[1] / 1e3
        out.append(f"| {k} | {grid} | {block} | {a[0]} | {a[1] / a[0]:.2f} | {a[1] / total * 100:.1f} % | {a[2] / a[0] / 1e6:.2f} | {a[3] / a[0] / 1e6:.2f} | {gbs:.0f} | {gbs / 6551:.2f} |")
    with open(os.path.join(PROF, name.replace(".csv", ".md")), "w") as fh:
        fh.write("\n".join(out) + "\n")
    return agg


def full_capture(rep, label, traffic_key, traffic, note="cold cache (ncu default cache control)"):
    src = os.path.join(OUT, rep)
    exported = src.replace(".ncu-rep", "_raw.csv")  # `ncu -i ... --page raw --csv` run on the GPU box (reports over
    if os.path.exists(src):                          # 32 MB do not fit gpurun's return channel next to each other)
        raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    elif os.path.exists(exported):
        raw = open(exported).read()
    else:
        return
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = [f"ncu --set full --clock-control none --import-source on ({rep}), {note}", ""]
    total = []
    for r in rows[2:]:
        out.append(f"kernel {r[hdr.index('Kernel Name')][:80]}  grid {r[hdr.index('Grid Size')]}  block {r[hdr.index('Block Size')]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                out.append(f"   {w:78s} {r[i]:>16s} {units[i]}")
        rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        total.append(rd * scale[units[hdr.index("dram__bytes_read.sum")]] + wr * scale[units[hdr.index("dram__bytes_write.sum")]])
        out.append("")
    with open(os.path.join(PROF, label), "w") as fh:
        fh.write("\n".join(out) + "\n")
    if total and traffic_key:
        traffic.setdefault(traffic_key[0], {})[traffic_key[1]] = sum(total) / len(total)


def main():
    os.makedirs(PROF, exist_ok=True)
    launch_list("r01_launches_hpcg192.csv", "hpcg192 (192^3, 4 levels)")
    launch_list("r01_launches_hpcg104.csv", "hpcg104 (104^3, 4 levels)")
    launch_list("r02_launches_hpcg192.csv", "hpcg192 (192^3, 4 levels), round 2")
    launch_list("r02_launches_hpcg104.csv", "hpcg104 (104^3, 4 levels), round 2")
    live_list("r02_iter_live_192.csv", "hpcg192 (192^3, 4 levels), round 2")
    live_list("r02_iter_live_104.csv", "hpcg104 (104^3, 4 levels), round 2")
    traffic = {}
    tpath = os.path.join(PROF, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    full_capture("r01_prof_gs_192.ncu-rep", "r01_ncu_gs_color_192.txt", ("gs_color_step_plain", "192x192x192"), traffic)
    full_capture("r01_prof_spmv_192.ncu-rep", "r01_ncu_spmv_192.txt", ("spmv_plain", "192x192x192"), traffic)
    # the dictionary-coded kernels (packed.cu): what bench.py's roofline.traffic reads
    full_capture("r01_gs_packed_192.ncu-rep", "r01_ncu_gs_packed_192.txt", ("gs_color_step", "192x192x192"), traffic)
    full_capture("r01_spmv_packed_192.ncu-rep", "r01_ncu_spmv_packed_192.txt", ("spmv", "192x192x192"), traffic)
    # the one-launch sweep of a small level (sweep_cluster.cu), eager launch of tools/cluster_sweep_once.py
    full_capture("r01_gs_sweep_8.ncu-rep", "r01_ncu_gs_sweep_8.txt", ("gs_sweep", "8x8x8"), traffic)
    full_capture("r01_gs_sweep_13.ncu-rep", "r01_ncu_gs_sweep_13.txt", ("gs_sweep", "13x13x13"), traffic)
    # round 2: the matrix-free plane kernels, live caches (--cache-control none)
    live = "live caches (--cache-control none): the traffic of the kernel inside a running sweep"
    full_capture("r02_planes_192.ncu-rep", "r02_ncu_planes_192.txt", ("gs_planes_launch", "192x192x192"), traffic, live)
    full_capture("r02_spmv_192.ncu-rep", "r02_ncu_spmv_planes_192.txt", ("spmv_planes", "192x192x192"), traffic, live)
    full_capture("r02_vector_192.ncu-rep", "r02_ncu_vector_192.txt", None, traffic, live)
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
