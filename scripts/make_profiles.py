"""Summarise a measurement pass (scripts/gpu_round.sh) into profiles/ (tracked).

    python scripts/make_profiles.py <tag>     # reads gpurun_out/*_<tag>*, writes profiles/<tag>_*

Writes:
  profiles/<tag>_launches.csv           per-kernel launch list summary (ncu gpu__time_duration, cold)
  profiles/<tag>_ncu_kernels.json       key `--set full` metrics per captured kernel
  profiles/ncu_sampler_summary.json     dram bytes per sampler launch (bench.py `roofline.traffic`)
  profiles/<tag>_bench.json             the bench line
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "scripts"))
from ncu_summary import load  # noqa: E402


def launches(tag):
    src = REPO / "gpurun_out" / f"launches_c3_{tag}.csv"
    rows = list(csv.reader(open(src)))
    # ncu --csv launch list: find header row
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        val = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        ms = val * scale
        agg[name][0] += 1
        agg[name][1] += ms
        seq.append((name, ms))
    out = REPO / "profiles" / f"{tag}_launches.csv"
    with open(out, "w") as f:
        f.write("kernel,launches,total_ms,share_pct\n")
        tot = sum(v[1] for v in agg.values())
        for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{name},{n},{ms:.3f},{100 * ms / tot:.1f}\n")
    return out


def capture_algorithmic_bytes(tag):
    """SURVEY §8(d) sampler bytes of the captured launch (iteration 13 of the ncu'd profile_run,
    whose log prints entries/T per iteration): T*18 + 4*sum(len*nnz) + 8*K*U."""
    log = REPO / "gpurun_out" / f"prof_sampler_c3_{tag}.log"
    if not log.exists():
        return None
    import re
    sys.path.insert(0, str(REPO))
    import bench
    cfg = bench.CONFIGS["c3"]
    et, units = None, None
    for line in log.read_text().splitlines():
        m = re.match(r"iter 13: .* entries/T=([0-9.]+)", line)
        if m:
            et = float(m.group(1))
        m = re.search(r"'num_units': (\d+)", line)
        if m:
            units = int(m.group(1))
    if et is None or units is None:
        return None
    return bench.sampler_bytes(cfg["T"], int(et * cfg["T"]), cfg["K"], units)


def kernels(tag):
    out = []
    for rep in (f"prof_sampler_c3_{tag}.ncu-rep", f"prof_sscphi_c3_{tag}.ncu-rep"):
        p = REPO / "gpurun_out" / rep
        if p.exists():
            out += load(str(p))
    keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
            "launch__block_size", "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]
    slim = [{k: kk[k] for k in ["name"] + [m for m in keep if m in kk] + [m + "@unit" for m in keep if m in kk]}
            for kk in out]
    # The evidence the north star asks for, per kernel: achieved DRAM GB/s (bytes moved / time,
    # under ncu), warp execution efficiency (active threads per issued instruction / 32) and
    # shared-memory bank conflicts.
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    for k in slim:
        try:
            byts = sum(k[m] * scale.get(k.get(m + "@unit", "byte"), 1) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            secs = k["gpu__time_duration.sum"] * tscale.get(k.get("gpu__time_duration.sum@unit", "ms"), 1e-3)
            k["derived_dram_gbs"] = byts / secs / 1e9
            k["derived_warp_exec_efficiency"] = k["smsp__thread_inst_executed_per_inst_executed.ratio"] / 32.0
        except (KeyError, ZeroDivisionError):
            pass
    (REPO / "profiles" / f"{tag}_ncu_kernels.json").write_text(json.dumps(slim, indent=1))
    for k in slim:
        if "sampler" in k["name"]:
            def gb(m):
                u = k.get(m + "@unit", "byte")
                f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
                return k[m] * f
            alg = capture_algorithmic_bytes(tag)
            dram = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
            summary = {"dram_bytes_per_launch": dram,
                       "algorithmic_bytes_at_capture": alg,
                       "dram_over_algorithmic": dram / alg if alg else None,
                       "dram_read_bytes": gb("dram__bytes_read.sum"), "dram_write_bytes": gb("dram__bytes_write.sum"),
                       "duration_ms_under_ncu": k["gpu__time_duration.sum"],
                       "config": f"C3 iteration 13 (steady state, as the bench), tag {tag}, ncu --set full --clock-control none"}
            (REPO / "profiles" / "ncu_sampler_summary.json").write_text(json.dumps(summary, indent=1))
    return slim


def main():
    tag = sys.argv[1]
    (REPO / "profiles").mkdir(exist_ok=True)
    print(launches(tag).read_text())
    for k in kernels(tag):
        print(k["name"], {m: k[m] for m in k if not m.endswith("@unit") and m != "name"})
    b = REPO / "gpurun_out" / f"bench_{tag}.json"
    if b.exists():
        (REPO / "profiles" / f"{tag}_bench.json").write_text(b.read_text())


if __name__ == "__main__":
    main()
