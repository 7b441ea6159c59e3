import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess, numpy as np
import paper_1209_2137_b200 as P
from tests.page_builder import build_fastpfor_page
from tests.test_collisions import blocks_for
if len(sys.argv) < 2:
    for kind in range(6):
        r = subprocess.run([sys.executable, __file__, str(kind)], capture_output=True, text=True)
        print(kind, (r.stdout.strip() or r.stderr.strip()[-150:]))
    sys.exit(0)
kind = int(sys.argv[1])
rng = np.random.default_rng(5)
bl = [b for i, b in enumerate(blocks_for(rng, 24)) if i % 6 == kind]
page, expect = build_fastpfor_page(bl, vertical=False)
codec = P.make_codec("fastpfor")
enc = P.layout(codec, [page], [len(expect)])
b = P.DeviceBatch(codec, enc, raw=True, indexed=False)
try:
    b.decode()
    print("status", b.statuses(), "eq", np.array_equal(b.output(), expect), [(x[1], x[2], len(x[3])) for x in bl])
except Exception as e:
    print("EXC", str(e)[:50], [(x[1], x[2], len(x[3])) for x in bl])
