# ncu --set full of one mid-sort k_onesweep pass of the C4 build; stall reasons + per-line table (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-os}
N=${N:-100000000} BUILDS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_onesweep}" -s ${SKIP:-5} -c 1 -o gpurun_out/prof_$TAG python tools/c4_build.py > gpurun_out/ncu_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_$TAG.txt
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv
python - <<PY
import csv
rows = list(csv.reader(open("gpurun_out/raw_$TAG.csv")))
h, u, v = rows[0], rows[1], rows[2]
for k, x in zip(h, v):
    if ("pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued")) or k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"):
        try:
            if float(x.replace(",", "")) == 0: continue
        except ValueError: pass
        print(k, x)
PY
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$TAG.csv 2>/dev/null
SORT=stall python tools/ncu_lines.py gpurun_out/src_$TAG.csv 45 > gpurun_out/lines_$TAG.txt; cat gpurun_out/lines_$TAG.txt
rm -f gpurun_out/src_$TAG.csv
