"""Summarise ncu artefacts into the text files committed under profiles/.

  python tools/ncu_summary.py launches <launches.csv> > profiles/rNN_launches.md
  python tools/ncu_summary.py report <x.ncu-rep> [algorithmic-bytes] > profiles/rNN_x.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*", "", name) if not name.startswith("void lmep") else name
    return name[:110]


def launches(path):
    rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(path) if l.startswith('"'))))]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    total = 0.0
    for r in rows[1:]:
        t = float(r[iv]) / 1e3
        k = short(r[ik])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
        total += t
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none)\n")
    print(f"source: `{path}`; {sum(a[0] for a in agg.values())} launches, {total:.1f} us total "
          f"(cold-cache, serialised by ncu: compare shares, not absolutes)\n")
    print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / total:.1f}% | {t / n:.2f} |")


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "dram bytes read"),
    ("dram__bytes_write.sum", "dram bytes write"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "thread DFMA"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "thread DADD"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "thread DMUL"),
]


def report(path, algo_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units, v = r[0], r[1], r[2]
    d = {k: (x, u) for k, u, x in zip(h, units, v)}
    kname = d.get("Kernel Name", ("?", ""))[0]
    print(f"# ncu --set full: `{kname}`\n\nsource: `{path}`\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k, lab in WANT:
        if k in d:
            print(f"| {lab} (`{k}`) | {d[k][0]} | {d[k][1]} |")
    stalls = []
    for k, (x, u) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(x), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("\nTop stall reasons (warps stalled per issued instruction):\n")
    for x, k in sorted(stalls, reverse=True)[:6]:
        print(f"- {k}: {x:.2f}")
    if algo_bytes:
        try:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * scale.get(d["dram__bytes_read.sum"][1], 1) + \
                wr * scale.get(d["dram__bytes_write.sum"][1], 1)
            print(f"\nDRAM traffic {tot:.4g} B vs algorithmic {float(algo_bytes):.4g} B "
                  f"(ratio {tot / float(algo_bytes):.3f})")
        except (KeyError, ValueError):
            pass


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
