# developer sweep of the SIMD-BP128 group kernel: tools/group_ab.sh "kw list" (0 = auto)
for g in $1; do
  echo "== IZG_GROUP=$g"
  if [ $g = 0 ]; then unset IZG_GROUP; else export IZG_GROUP=$g; fi
  IZG_SPLIT=0 timeout 600 python tools/split_sweep.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    if 'bp128' in d['codec']: print(d['codec'], d['chunks'], 'no-ws path (group/one-warp)', d['one_warp_ms'], d['ws_path_ok'])"
done
unset IZG_GROUP
