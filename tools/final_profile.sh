# Round-end evidence for profiles/ (run on the GPU box via gpurun):
#   launch list of the bench command (gpu__time_duration per launch), one
#   ncu --set full capture of each kernel of the C5 step, at full size.
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python bench.py --steps 20 --warmup 5 > $OUT/bench.log 2>&1
tail -1 $OUT/bench.log
$NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
echo launches rc=$?
$NCU --set full --import-source on --clock-control none -k regex:"decode_kernel|fp_index|fp_team" -s 3 -c 3 \
    -o $OUT/c5_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo full rc=$?
