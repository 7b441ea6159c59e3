# Round-end evidence, last session of round 2 (run on the GPU box via gpurun):
# GPU suite, smoke, the bench lines (C5 default, C1, C4, reference arm), the
# launch list of the bench command and one full ncu capture of each kernel of
# the C5 step.
set -x
OUT=gpurun_out/final3
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
PYTHONUNBUFFERED=1 timeout -s KILL 1500 python -u -m pytest tests -m gpu -q > $OUT/gputests.log 2>&1; tail -3 $OUT/gputests.log > $OUT/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 300 python bench.py --workload c1 --no-cpu-baseline > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 300 python bench.py --workload c4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none -k regex:"decode_kernel|fp_index|fp_team" -s 3 -c 3 -o $OUT/c5_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
tail -2 $OUT/gputests.txt; cat $OUT/smoke.txt | tail -1; tail -c 600 $OUT/bench_c5.json
