bash tools/final_run.sh
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"decode_kernel|fp_index" -c 3 -o gpurun_out/final/c5_full python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/final/c5_full.log 2>&1
