# developer A/B: tools/ab.sh "variantA variantB ..." "quick_bench configs"
for v in $1; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  echo "== $v"; timeout 300 python tools/quick_bench.py $2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['name'], d['model'], d['d'], d['rate'], d['ok'], d['ms'], d['gints'], d['frac'])"
done
