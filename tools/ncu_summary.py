"""Summarise ncu captures into profiles/ (text, tracked in git).

    python tools/ncu_summary.py report <file.ncu-rep> [--algo-bytes B]   # one --set full capture
    python tools/ncu_summary.py launches <launches.csv>                  # gpu__time_duration list
"""
import csv
import subprocess
import sys
from collections import OrderedDict

KEYS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU data-pipe wavefronts % (MIO: LDS/STS/SHFL/STG)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-pipe wavefronts (LDS+STS+SHFL)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "CTA limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (shared mem)"),
])
STALLS = ["short_scoreboard", "math_pipe_throttle", "wait", "not_selected", "dispatch_stall", "mio_throttle",
          "long_scoreboard", "lg_throttle", "barrier", "no_instruction", "selected"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def report(rep, algo_bytes=None):
    h, units, rows = raw(rep)
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", ""]
    for row in rows:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        lines.append(f"## {d.get('Kernel Name', '?')}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k, name in KEYS.items():
            if k in d:
                lines.append(f"| {name} (`{k}`) | {d[k]} | {u.get(k, '')} |")
        w = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        r = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wu, ru = u.get("dram__bytes_write.sum", ""), u.get("dram__bytes_read.sum", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = w * scale.get(wu, 1) + r * scale.get(ru, 1)
        lines.append(f"| **traffic = read + write** | {traffic:.6g} | byte |")
        if algo_bytes:
            lines.append(f"| algorithmic bytes (4 B/sample) | {algo_bytes:.6g} | byte |")
            lines.append(f"| traffic / algorithmic | {traffic / algo_bytes:.5f} | |")
        lines.append("")
        lines.append("Warp stall reasons (warps per issue-active cycle):")
        lines.append("")
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d:
                lines.append(f"- {s}: {d[k]}")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = OrderedDict(), {}
    for r in rows[1:]:
        k = r[ik].split("(")[0]
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[iu], 1.0)
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] = cnt.get(k, 0) + 1
    T = sum(tot.values())
    lines = [f"# launch list summary: `{path.split('/')[-1]}` (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        lines.append(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / T:.1f}% |")
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1] == "report":
        ab = float(sys.argv[sys.argv.index("--algo-bytes") + 1]) if "--algo-bytes" in sys.argv else None
        print(report(sys.argv[2], ab))
    else:
        print(launches(sys.argv[2]))
