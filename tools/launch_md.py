"""Markdown table of the last matvec's launches from an ncu
--metrics gpu__time_duration.sum --csv log (dev tool)."""
import csv
import re
import sys


def table(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    recs = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()
        if name.startswith("at::"):   # the driver script's own checksum kernels
            continue
        recs.append((name, r[gi] if gi is not None else "", us))
    starts = [i for i, rec in enumerate(recs) if "permute_in" in rec[0] or "prologue_kernel" in rec[0] or "upward8" in rec[0] or "upward_cube" in rec[0]]
    last = recs[starts[-1]:] if starts else recs
    tot = sum(x[2] for x in last)
    out = [f"## {title}: one matvec = {tot:.1f} us of kernel time", "", "| kernel | grid | us | share |",
           "|---|---|---|---|"]
    for name, grid, us in last:
        out.append(f"| `{name}` | {grid} | {us:.1f} | {100 * us / tot:.1f}% |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    for i in range(0, len(args), 2):
        print(table(args[i], args[i + 1]))
