mkdir -p gpurun_out/final
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/final/bench_c1.json 2> gpurun_out/final/bench_c1.err
timeout 300 ncu --set full --clock-control none -k regex:split_kernel -c 1 -o gpurun_out/final/split_bp_64 python tools/profile_small.py simdbp128-s4 64 2 > /dev/null 2>&1
IZG_NOWS=1 timeout 300 ncu --set full --clock-control none -k regex:group_kernel -c 1 -o gpurun_out/final/group_bp_64 python tools/profile_small.py simdbp128-s4 64 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:split_kernel -c 1 -o gpurun_out/final/split_fp_64 python tools/profile_small.py simdfastpfor-s4 64 2 > /dev/null 2>&1
ls gpurun_out/final
