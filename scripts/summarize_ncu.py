"""Summarise ncu output into profiles/ (run here, no GPU needed).

  python scripts/summarize_ncu.py full   <report.ncu-rep> [units_per_launch]  -> markdown on stdout
  python scripts/summarize_ncu.py launch <launches.csv>                        -> markdown on stdout

`full` reads `ncu -i ... --page raw --csv` and `--page source --csv` of a
`--set full` capture; `launch` reads the CSV of a
`--metrics gpu__time_duration.sum` launch list (cold-cache, serialised:
compare shares, not absolute times).
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def _ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def full(rep, units=None):
    rows = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "raw", "--csv"]))))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (v[i], u[i]) for i, k in enumerate(h)}
    out = [f"### `{d.get('Kernel Name', ('?',))[0]}`", "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in d:
            out.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
    rd = float(d["dram__bytes_read.sum"][0]) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
    wr = float(d["dram__bytes_write.sum"][0]) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
    out.append(f"| dram bytes read+write (per launch) | {rd + wr:.0f} | byte |")
    st = [(k, float(val)) for k, (val, _) in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and val not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    out += ["", "Top stall reasons (warps per issued instruction):", ""]
    out += [f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: "
            f"{x:.3f}" for k, x in st[:8]]
    src = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        sh = src[1]
        iS, iT = sh.index("Source"), sh.index("Thread Instructions Executed")
        cnt = collections.Counter()
        for r in src[2:]:
            try:
                e = float(r[iT] or 0)
            except (ValueError, IndexError):
                continue
            toks = r[iS].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            cnt[op.split(".")[0]] += e
        tot = sum(cnt.values())
        if units:
            out += ["", f"SASS thread-instructions per unit ({units:.0f} units per launch): {tot / units:.1f}", ""]
            out += [f"- {op}: {e / units:.2f}" for op, e in cnt.most_common(14)]
            fp64 = sum(cnt[o] for o in ("DFMA", "DMUL", "DADD")) / units
            out.append(f"- FP64 (DFMA+DMUL+DADD): {fp64:.2f} per unit")
    out.append("")
    return "\n".join(out), rd + wr


def launch(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:90]
        agg[short][0] += 1
        agg[short][1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(t for _, t in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "full":
        md, _ = full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
        print(md)
    else:
        print(launch(sys.argv[2]))
