"""Writes the committed profile summaries from one gpurun capture (run here,
after the bench / ncu commands of DESIGN §5 wrote gpurun_out/): the bench
line, the reference arm, the launch list + summary, the k_manifold ncu
details + instruction mix + stalls, and profiles/kernel_traffic.json.
Usage: python tools/refresh_profiles.py <tag> [prefix]   (e.g. r2 r2)
With gpurun_out/batch_fit_<tag>.ncu-rep present, also writes
profiles/<prefix>_ncu_batch_fit.txt (lattice assembly, flow Cholesky, flow
band solve)."""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def batch_fit_summary(rep, dst):
    raw = list(csv.reader(subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    hdr, units = raw[0], raw[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "lts__t_sector_hit_rate.pct"]
    lines = ["ncu --set full --clock-control none, one launch each (C5 batch ridge: 10^7 points,",
             "99,856 lattice centres, band ld 2912) of python tools/time_batch_c5.py", ""]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", "")[:60]
        lines.append(name)
        for k in want:
            if k in d:
                lines.append(f"  {k:64s} {d[k]:>14s} {units[hdr.index(k)]}")
    dst.write_text("\n".join(lines) + "\n")


def main(tag, prefix="r1"):
    rep = OUT / f"batch_fit_{tag}.ncu-rep"
    if rep.exists():
        batch_fit_summary(rep, PROF / f"{prefix}_ncu_batch_fit.txt")
    shutil.copy(OUT / f"bench_{tag}.json", PROF / f"{prefix}_bench.json")
    shutil.copy(OUT / f"bench_ref_{tag}.json", PROF / f"{prefix}_bench_reference_arm.json")
    shutil.copy(OUT / f"launches_{tag}.csv", PROF / f"{prefix}_bench_launches.csv")
    summ = subprocess.run([sys.executable, str(ROOT / "tools" / "summarize_launches.py"),
                           str(OUT / f"launches_{tag}.csv"),
                           "python bench.py --steps 2 --warmup 3 --no-cpu"],
                          capture_output=True, text=True, check=True).stdout
    (PROF / f"{prefix}_bench_launches_summary.csv").write_text(summ)
    rep = str(OUT / f"bench_manifold_{tag}.ncu-rep")

    def ncu(*args):
        return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout

    details = ncu("--page", "details")
    raw = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
    d = dict(zip(raw[0], raw[2]))
    units = dict(zip(raw[0], raw[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units["dram__bytes_read.sum"]]
    f = lambda k: float(d[k])  # noqa: E731
    traffic = {"k_manifold": {
        "points": 10_000_000,
        "dram_bytes_per_launch": (f("dram__bytes_read.sum") + f("dram__bytes_write.sum")) * scale,
        "dram_read_bytes": f("dram__bytes_read.sum") * scale,
        "dram_write_bytes": f("dram__bytes_write.sum") * scale,
        "algorithmic_bytes": 810_000_000,
        "kernel_us_under_ncu": f("gpu__time_duration.sum"),
        "fp64_pipe_pct_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "l1_lsu_wavefronts_pct_elapsed":
            f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "source": "ncu --set full --clock-control none, one k_manifold launch of python bench.py "
                  "--steps 2 --warmup 3 --no-cpu --no-update; details in "
                  f"profiles/{prefix}_ncu_k_manifold_full.txt"}}
    (PROF / "kernel_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    src = list(csv.reader(ncu("--page", "source", "--csv", "--print-source", "sass").splitlines()))
    hdr = src[1]
    ix = {h: i for i, h in enumerate(hdr)}
    agg, tot = collections.defaultdict(float), 0.0
    for r in src[2:]:
        s = r[ix["Source"]].strip()
        if not s:
            continue
        t = s.split()
        op = t[1] if t[0].startswith("@") else t[0]
        v = float(r[ix["Instructions Executed"]] or 0)
        agg[op] += v
        tot += v
    warps = 10_000_000 / 32
    lines = ["", "Instruction mix (SASS, warp-level instructions per 32 points):",
             f"  total {tot / warps:.1f}"]
    lines += [f"  {k:28s} {v / warps:8.1f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:25]]
    stalls = sorted(((float(v), h) for h, v in d.items()
                     if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")
                     and v not in ("", "0")), reverse=True)[:8]
    lines += ["Warp stall samples (top):"] + [f"  {v:10.0f} {h}" for v, h in stalls]
    (PROF / f"{prefix}_ncu_k_manifold_full.txt").write_text(details + "\n".join(lines) + "\n")
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
