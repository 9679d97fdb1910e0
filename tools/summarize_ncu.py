"""Compact summary of ncu --set full reports (key metrics + top stall reasons) as markdown."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def summarize(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else rep
    out = [f"### {name.split('(')[0]}  (`{rep}`)", "", "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out.append(f"| {label} (`{k}`) | {vals[i]} {units[i]} |")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(vals[i]), h.split("stalled_")[1]))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    out.append("")
    out.append("top stall reasons (pc samples): " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:6]))
    out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n".join(summarize(r) for r in sys.argv[1:]))
