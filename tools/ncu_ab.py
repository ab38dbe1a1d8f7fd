"""Summarise ncu --csv metric dumps (tools A/B runs): one line per file."""
import csv
import glob
import sys

for f in sorted(sum((glob.glob(a) for a in sys.argv[1:]), [])):
    lines = open(f).read().splitlines()
    try:
        i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    except IndexError:
        print(f, "no data")
        continue
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    mi, vi = h.index("Metric Name"), h.index("Metric Value")
    d = {r[mi]: float(r[vi].replace(",", "")) for r in rows[1:]}
    at = d.get("smsp__inst_executed_op_shared_atom.sum", 0.0)
    aw = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 0.0)
    print(f.split("/")[-1], "inst %.2fe9 atoms %.2fe9 atom_wf %.2fe9 (%.2f/inst, conflicts %.2fe9) ld_wf %.2fe9 "
          "issue %.0f%% dur %.1f ms" % (d["smsp__inst_executed.sum"] / 1e9, at / 1e9, aw / 1e9, aw / max(at, 1),
                                          d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", 0) / 1e9,
                                          d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 0) / 1e9,
                                          d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
                                          d["gpu__time_duration.sum"] / 1e6))
