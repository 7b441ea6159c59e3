# developer A/B of the fused page kernels: tools/fused_ab.sh "variants"
for v in $1; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  echo "== $v"; IZG_FUSED=1 timeout 300 python tools/quick_bench.py c5fp c4 | cut -c1-200; timeout 300 python tools/f3_bench.py 2>&1 | grep -E "fastpfor-s4|simplepfor" | cut -c1-160
  CODEC=simdfastpfor-s4 timeout 300 python tools/intersect_bench.py 2>&1 | tail -1 | cut -c1-200
done
