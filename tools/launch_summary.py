"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv profiles/<name>.txt "<header>"
"""
import collections
import csv
import sys


def main(src, dst, header=""):
    rows = [r for r in csv.reader(open(src)) if r]
    head_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head_i]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.OrderedDict()
    for r in rows[head_i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].strip()
        ns = float(r[iv].replace(",", ""))
        cnt, t = tot.get(name, (0, 0.0))
        tot[name] = (cnt + 1, t + ns)
    unit = h[h.index("Metric Unit")] if "Metric Unit" in h else ""
    lines = [header, ""] if header else []
    for name, (cnt, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:74]:76s}{cnt:4d} launches {t / 1e6:12.3f} ms")
    open(dst, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
