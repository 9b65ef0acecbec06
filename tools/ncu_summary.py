"""Summarise an ncu report: per kernel duration, DRAM bytes/throughput, FP64 pipe,
warps active, top stall reasons, and (with --sass) the opcode mix.
python tools/ncu_summary.py report.ncu-rep [--sass]"""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for r in rows[2:]:
    print("==", r[col["Kernel Name"]])
    for w in want:
        if w in col:
            print(f"   {w:62s} {r[col[w]]:>16s} {units[col[w]]}")
    st = []
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{h} {v / tot * 100:.0f}%" for v, h in st[:6]))
if "--sass" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = list(csv.reader(io.StringIO(src)))
    k = None
    for i, l in enumerate(lines):
        if l and l[0] == "Kernel Name":
            if k is not None:
                break
            k = i
    hdr = lines[k + 1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ex, stl = Counter(), Counter()
    for l in lines[k + 2:]:
        if len(l) <= iE or (l and l[0] == "Kernel Name"):
            break
        toks = l[iS].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        try:
            ex[op] += int(l[iE]); stl[op] += int(l[iW])
        except ValueError:
            pass
    tot, ts = sum(ex.values()) or 1, sum(stl.values()) or 1
    for op, v in ex.most_common(14):
        print(f"   {op:10s} {v / tot * 100:5.1f}% inst {stl[op] / ts * 100:5.1f}% stall")
