"""Summarise ncu reports / launch lists into markdown for profiles/.

    python tools/summarize_ncu.py report.ncu-rep [...]        # --set full captures
    python tools/summarize_ncu.py --launches launches.csv     # gpu__time_duration list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, r, units)}


def summarize(rep):
    lines = [f"### `{rep}`", ""]
    for rec in raw(rep):
        name = rec.get("Kernel Name", ("?", ""))[0]
        lines.append(f"**{name[:110]}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in KEYS:
            if key in rec:
                v, u = rec[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"][:100]][0] += 1
            agg[d["Kernel Name"][:100]][1] += float(d["Metric Value"])
    tot = sum(t for _, t in agg.values())
    out = ["| launches | total ms | share | kernel |", "|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% | `{n}` |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
