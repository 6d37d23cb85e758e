"""Summarise ncu outputs brought back from gpurun into profiles/.

    python scripts/ncu_summary.py launches <launches.csv> <out.md>
    python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [--alg-bytes NAME=BYTES ...]

`launches`: per-kernel-name launch count, total / mean device time and the
share of the summed device time (cold-cache, serialised: compare shares).
`full`: the key metrics of every captured launch (duration, DRAM bytes,
throughputs, occupancy, registers, fp64 pipe) plus, if given, the
algorithmic bytes per launch and DRAM traffic / algorithmic ratio.
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def short(name):
    return name.split("(")[0].replace("void ", "")[:110]


def launches(path, out):
    agg = collections.OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"])
        if r.get("Metric Unit") == "us":
            v *= 1e3
        elif r.get("Metric Unit") == "ms":
            v *= 1e6
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        f.write(f"{sum(a[0] for a in agg.values())} launches, {tot/1e6:.3f} ms summed device time "
                "(cold-cache, serialised; compare shares)\n\n")
        f.write("| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|\n")
        for k, (n, t) in rows:
            f.write(f"| `{k}` | {n} | {t/1e6:.3f} | {t/n/1e3:.2f} | {t/tot:.4f} |\n")
    print(open(out).read())


def full(path, out, alg):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for key, nm in KEYS:
            if key in hdr:
                i = hdr.index(key)
                d[nm] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({path})\n\n")
        for d in res:
            f.write(f"## `{d['kernel']}`\n\n")
            for k, v in d.items():
                if k != "kernel":
                    f.write(f"* {k}: {v}\n")
            for nm, b in alg.items():
                if nm in d["kernel"]:
                    def mb(s):
                        v, u = s.split()
                        return float(v.replace(",", "")) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
                                                            "Gbyte": 1e3}.get(u, 1.0)
                    tr = mb(d["dram_read"]) + mb(d["dram_write"])
                    f.write(f"* algorithmic bytes per launch: {b/1e6:.1f} MB; DRAM traffic {tr:.1f} MB "
                            f"(ratio {tr/(b/1e6):.3f})\n")
            f.write("\n")
    print(open(out).read())
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        alg = {}
        for a in sys.argv[4:]:
            if "=" in a:
                k, v = a.split("=")
                alg[k] = float(v)
        full(sys.argv[2], sys.argv[3], alg)
