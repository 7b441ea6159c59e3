# CTA kernel variants A/B (developer tool): bash tools/cta_ab.sh "default v1 v2" "c1 c1big"
export IZG_CTA=1
for v in $1; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  echo "== $v"; timeout 200 python tools/quick_bench.py $2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['name'], d['model'], d['d'], d['ok'], d['ms'], d['gints'], d['frac'])"
done
