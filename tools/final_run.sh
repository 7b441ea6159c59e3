set -x
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_c5.json 2> gpurun_out/final/bench_c5.err
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/final/bench_c1.json 2> gpurun_out/final/bench_c1.err
timeout 300 python bench.py --workload c4 --no-cpu-baseline > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final/ncu_launch.log 2>&1
