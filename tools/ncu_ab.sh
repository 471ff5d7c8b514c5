#!/bin/bash
# A/B: key ncu metrics of the sweep kernel for two library builds (libA.so, libB.so in gpurun_out/ab/)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_wait"
for v in A B; do
  cp ab/lib$v.so paper_cs_0412107_b200/libmcinv.so
  touch paper_cs_0412107_b200/libmcinv.so
  timeout 200 python tools/run_one.py --config 2 --sweeps 6 --burn 1 > gpurun_out/ab_plain_$v.log 2>&1 &&
  timeout 600 ncu --metrics $M -k regex:"sweep[34]" -c 1 --csv python tools/run_one.py --config 2 --sweeps 6 --burn 1 > gpurun_out/ab_$v.csv 2>&1
  for r in 1 2; do timeout 200 python tools/run_one.py --config 2 --sweeps 22 --repeat 2 2>&1 | tail -1 >> gpurun_out/ab_time_$v.log; done
done
