"""Summarise an ncu report: key metrics per kernel (details page) and stall reasons (raw)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
want = ["Duration", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Issue Slots Busy",
        "Executed Ipc Active", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem", "Block Limit Registers"]
seen = set()
for row in r[1:]:
    key = (row[ki][:48], row[mi])
    if row[mi] in want and key not in seen:
        seen.add(key)
        print(f"{row[ki][:48]:48s} | {row[mi]} = {row[vi]} {row[ui]}")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units, rows = r[0], r[1], r[2:]
keys = ["smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed_op_shared_atom.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
for row in rows:
    name = row[hdr.index("Kernel Name")][:40]
    vals = {k: row[hdr.index(k)] for k in keys if k in hdr}
    print(name, vals)
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(row[i].replace(",", "") or 0))
          for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    st.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in st)
    print("   stalls:", ", ".join(f"{k} {v / tot:.0%}" for k, v in st[:6]))
