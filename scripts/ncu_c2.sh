#!/bin/bash
# ncu metrics of the c2 solve kernel (one launch): time, instructions, IPC, stalls.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 ncu --clock-control none -k regex:k_solve_fx -c 1 -s 2 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,launch__registers_per_thread,dram__bytes_read.sum,smsp__average_warp_latency_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_wait,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct,smsp__warp_issue_stalled_not_selected_per_warp_active.pct,smsp__warp_issue_stalled_selected_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_no_instruction_per_warp_active.pct,smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct \
  python bench.py --config ${2:-c2} --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$TAG.txt 2>&1
grep -E "k_solve|duration|inst_exec|per_cycle|registers|dram|stalled" gpurun_out/ncu_$TAG.txt | head -40
