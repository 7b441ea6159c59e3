# developer A/B under ncu: tools/ncu_ab.sh "variants" config
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_op_shfl.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio
mkdir -p gpurun_out
for v in $1; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  echo "== $v"
  timeout 300 ncu --clock-control none --metrics $M -k regex:"decode_kernel|fp_index" -c 2 --csv --log-file gpurun_out/ncu_ab_$v.csv python tools/profile_one.py $2 1 > /dev/null 2>&1
  python tools/ncu_csv.py gpurun_out/ncu_ab_$v.csv | sed 's/void izg:://'
done
