# developer sweep of the split kernel: tools/split_ab.sh "variants" ["segs list"]
for v in $1; do
  if [ $v = default ]; then unset IZG_LIB_PATH; else export IZG_LIB_PATH=$PWD/paper_1209_2137_b200/_lib/variants/$v.so; fi
  for sg in ${2:-0}; do
    echo "== $v segs=$sg"
    if [ $sg = 0 ]; then unset IZG_SPLIT_SEGS; else export IZG_SPLIT_SEGS=$sg; fi
    IZG_SPLIT=1 timeout 600 python tools/split_sweep.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['codec'], d['chunks'], d['ws_ms'], d['one_warp_ms'], d['ws_path_ok'])"
  done
done
unset IZG_SPLIT_SEGS
