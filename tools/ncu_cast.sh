#!/bin/bash
# Quick ncu metric capture of one k_cast launch of the C2 bench workload (run under gpurun).
# usage: tools/ncu_cast.sh <tag> [extra bench args]
tag=$1; shift
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__registers_per_thread,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_local_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum
ncu --metrics $M --clock-control none -k regex:k_cast -s 3 -c 1 --csv python bench.py --mode cast --steps 1 --warmup 2 --no-e2e --no-cpu "$@" > gpurun_out/ncu_$tag.csv 2> gpurun_out/ncu_$tag.err
python - "$tag" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = [r for r in csv.reader(l for l in open(f"gpurun_out/ncu_{tag}.csv") if l.startswith('"'))]
h = rows[0]
for r in rows[1:]:
    print(f"{tag:12s} {r[h.index('Metric Name')]:80s} {r[h.index('Metric Value')]}")
PY
