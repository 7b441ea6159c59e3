import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess, numpy as np, json
import paper_1209_2137_b200 as P
from tests.page_builder import build_fastpfor_page
cases = [(nb, pos, b, mb, vert) for nb in (1, 2, 4) for pos in ([77, 77], [77, 78], [5], [77])
         for (b, mb) in ((3, 9),) for vert in (False,)] + [(1, [77, 77], 3, 9, True), (1, [5], 0, 1, False), (1, [5], 3, 4, False), (1, [5, 6], 3, 4, False)]
if len(sys.argv) < 2:
    for i, c in enumerate(cases):
        r = subprocess.run([sys.executable, __file__, str(i)], capture_output=True, text=True)
        print(c, (r.stdout.strip() or r.stderr.strip()[-150:])[:60])
    sys.exit(0)
nb, pos, b, mb, vert = cases[int(sys.argv[1])]
low = np.arange(128, dtype=np.uint64) * 3
bl = [(low, b, mb, pos, [5 + k for k in range(len(pos))]) for _ in range(nb)]
page, expect = build_fastpfor_page(bl, vertical=vert)
codec = P.make_codec("simdfastpfor" if vert else "fastpfor")
enc = P.layout(codec, [page], [len(expect)])
b_ = P.DeviceBatch(codec, enc, raw=True, indexed=False)
try:
    b_.decode()
    print("ok" if np.array_equal(b_.output(), expect) else "WRONG", b_.statuses())
except Exception as e:
    print("EXC", str(e)[:40])
