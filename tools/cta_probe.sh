# CTA kernel A/B and profile (developer tool)
export IZG_CTA=1
for v in default nochain; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  echo "== $v"; timeout 120 python tools/quick_bench.py c1big 2>&1 | tail -1
done
unset IZG_LIB_PATH
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"cta_kernel" -s 1 -c 1 -o gpurun_out/r02_cta_c1big python tools/profile_one.py c1big 2 > /dev/null 2>&1
echo ncu rc=$?
