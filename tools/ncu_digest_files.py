"""Committed digest of one ncu --set full capture from its exported files (summary from
tools/ncu_summary.py, --page raw --csv, --page source --csv --print-source cuda,sass).
usage: ncu_digest_files.py SUMMARY RAW SRC ROWS "command" > profiles/...txt"""
import csv
import subprocess
import sys

summ, raw, src, rows, cmd = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5]
print(f"# ncu --set full --clock-control none --import-source on: {cmd}")
print(open(summ).read().rstrip())
r = list(csv.reader(open(raw)))
d = dict(zip(r[0], r[2]))
rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
unit_r, unit_w = r[1][r[0].index("dram__bytes_read.sum")], r[1][r[0].index("dram__bytes_write.sum")]
print(f"   dram__bytes_read.sum  {rd} {unit_r}")
print(f"   dram__bytes_write.sum {wr} {unit_w}")
st = []
for k, x in d.items():
    if "smsp__average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            st.append((float(x), k.split("stalled_")[1].split("_per")[0]))
        except ValueError:
            pass
print("   stall reasons (warps per issued instruction):",
      ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:9]))
for k in ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"):
    if k in d:
        print(f"   {k} {d[k]}")
print()
print("# executed warp-instructions per input row, top source lines (tools/ncu_bylines.py):")
sys.stdout.flush()
subprocess.run([sys.executable, "tools/ncu_bylines.py", src, str(int(rows)), "30"])
