"""Summarise an ncu --set full report (+ optional launch-list CSV) into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.md [--launches launches.csv] [--n 134217728]

Per kernel: duration, DRAM bytes read/written (the ``traffic`` figure of the
bench roofline), throughput, issue/warp activity, registers, top stall
reasons, and the executed/algorithmic byte ratio for the KKT matvec passes.
"""
import argparse
import csv
import io
import subprocess

ALG_PER_VOXEL = {  # algorithmic bytes per voxel of each launch of one KKT matvec
    "fast_pass": 16.0,
    "mirror_pass": 16.0,
    "split_pass": 16.0,
    "group_pass<512, 2": 16.125,
    "group_pass<1024, 2": 16.125,
    "k_kkt_epilogue": 56.0,
}


def raw_rows(rep):
    """Header, units and data rows of the raw page (an .ncu-rep, or the
    ``--page raw --csv`` export of one made on the GPU box)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
        out = out[out.index('"ID"'):] if '"ID"' in out else out
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--n", type=float, default=512.0 ** 3)
    a = ap.parse_args()
    hdr, units, data = raw_rows(a.report)
    col = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        return r[col[k]] if k in col else ""

    lines = [f"# ncu summary: `{a.report.split('/')[-1]}`", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | traffic/alg | DRAM % peak | issue active % | warps active % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in data:
        name = g(r, "Kernel Name")
        short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        short = short.replace("fl::<unnamed>::", "").replace("<unnamed>::", "")
        rd, wr = float(g(r, "dram__bytes_read.sum") or 0), float(g(r, "dram__bytes_write.sum") or 0)
        ru = units[col["dram__bytes_read.sum"]]
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(ru, 1.0)
        rd_gb, wr_gb = rd * scale, wr * scale
        alg = next((v for k, v in ALG_PER_VOXEL.items() if k in name), None)
        ratio = f"{(rd_gb + wr_gb) * 1e9 / (alg * a.n):.3f}" if alg else "-"
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {v:.1f}" for v, n in sorted(stalls, reverse=True)[:3])
        tu = units[col["gpu__time_duration.sum"]] if "gpu__time_duration.sum" in col else "msecond"
        ms = float(g(r, "gpu__time_duration.sum") or 0) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
                                                           "second": 1e3}.get(tu, 1.0)
        lines.append(f"| `{short[:60]}` | {ms:.4f} | {rd_gb:.3f} | {wr_gb:.3f} | {ratio} | "
                     f"{float(g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                     f"{float(g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                     f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                     f"{g(r, 'launch__registers_per_thread')} | {top} |")
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[start]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        per = {}
        for r in rows[start + 1:]:
            if len(r) <= vi or r[h.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = r[ki].split("(")[0].replace("void ", "")
            per.setdefault(k, []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        lines += ["", f"## Launch list (`{a.launches.split('/')[-1]}`, cold-cache serialised ncu timings)", "",
                  "| kernel | launches | total time | share |", "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
