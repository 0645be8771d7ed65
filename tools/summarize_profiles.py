"""Summarise an ncu launch list + full capture into markdown (profiles/)."""
import collections
import csv
import io
import subprocess
import sys


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault(d["Kernel Name"].split("(")[0], []).append(float(d["Metric Value"]) / 1000.0)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches/step | mean µs | µs/step | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v) / steps:g} | {sum(v) / len(v):.1f} | {sum(v) / steps:.1f} | {sum(v) / tot:.3f} |")
    out.append(f"| **total** | | | {tot / steps:.1f} | 1.000 |")
    return "\n".join(out)


WANT = [("gpu__time_duration.sum", "µs"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
        ("launch__registers_per_thread", "regs"), ("pcie__read_bytes.sum.per_second", "PCIe rd/s"),
        ("launch__grid_size", "grid")]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    idx = {w: hdr.index(w) for w, _ in WANT if w in hdr}
    out = ["| kernel | " + " | ".join(f"{lab} ({units[idx[w]]})" if w in idx else lab for w, lab in WANT) + " |",
           "|---" * (len(WANT) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        out.append(f"| `{name}` | " + " | ".join(r[idx[w]] if w in idx else "" for w, _ in WANT) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[1], int(sys.argv[2])))
    print()
    print(full(sys.argv[3]))
