"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, total time, share. Usage: summarize_launches.py launches.csv "command" > out.csv"""
import collections
import csv
import sys


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    h = next(rd)
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for r in rd:
        if r[im] == "gpu__time_duration.sum":
            name = r[ik]
            if "distribution_elementwise" in name:
                name = "torch::distribution_elementwise (synthetic input RNG)"
            rows.append((name.split("(")[0] if name.startswith(("tlg", "void tlg")) else name[:120],
                         float(r[iv].replace(",", "")) / 1e3))
    agg = collections.OrderedDict()
    for n, us in rows:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# ncu launch list summary: {cmd}")
    print("# (gpu__time_duration.sum, --clock-control none, serialized + cold caches: compare shares)")
    print(f"# {len(rows)} launches captured; total {tot / 1e3:.3f} ms")
    print("kernel,launches,total_us,share")
    for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"\"{n}\",{c},{us:.1f},{us / tot:.4f}")


if __name__ == "__main__":
    main()
