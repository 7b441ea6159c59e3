import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess, numpy as np
import paper_1209_2137_b200 as P
from tests.page_builder import build_fastpfor_page
if len(sys.argv) < 2:
    for off in range(8):
        for pad in (0, 64):
            r = subprocess.run([sys.executable, __file__, str(off), str(pad)], capture_output=True, text=True)
            print(off, pad, (r.stdout.strip() or r.stderr.strip()[-150:])[:50])
    sys.exit(0)
off, pad = int(sys.argv[1]), int(sys.argv[2])
low = np.arange(128, dtype=np.uint64) * 3
page, expect = build_fastpfor_page([(low, 3, 4, [5], [1])], vertical=False)
words = np.zeros(off + len(page) + 8 + pad, dtype=np.uint32)
words[off:off + len(page)] = page
table = np.zeros(1, dtype=P._native.CHUNK_DTYPE)
table[0] = (off, len(page), 128, 0)
codec = P.make_codec("fastpfor")
b_ = P.DeviceBatch(codec, P.Encoded(words, table), raw=True, indexed=False)
try:
    b_.decode()
    print("ok" if np.array_equal(b_.output(), expect) else "WRONG", b_.statuses())
except Exception as e:
    print("EXC", str(e)[:40])
try:
    import ctypes
    L = P._native.lib()
    buf = (ctypes.c_uint32 * 8)()
    print("dbg", L.izg_debug_read(buf), list(buf))
except Exception as e:
    print("dbg unavailable", e)
