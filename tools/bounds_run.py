"""Developer: the SIMD-FastPFOR fuzz / mutation / collision / heavy-page suites under the
bounds-check build (python tools/build_variant.py bounds -DIZG_BOUNDS), with the team decode
and both page index passes forced; prints the violation counters of the team decode and of
the index kernels.  This is the repository's own memcheck for the new round-2 kernels: the
pool refuses compute-sanitizer.

    IZG_LIB_PATH=.../variants/bounds.so python tools/bounds_run.py
"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SCRIPT = r'''
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_1209_2137_b200 as P
from oracle.pyoracle import Oracle, Reference
from tests import test_gpu_parity as T
from tests import test_gpu_indexed as TI
from tests import test_collisions as TC
from tests import test_gpu_team as TT
O, R = Oracle(), Reference()
for name in ["simdfastpfor", "simdfastpfor-s4", "simdfastpfor-d2", "simdfastpfor-dm"]:
    T.test_roundtrip_assorted(torch, O, name)
    for wp, op in [(1, 0), (2, 3), (0, 2), (3, 1)]:
        T.test_unaligned_placement(torch, name, wp, op)
    T.test_mutation_fuzz_matches_oracle(torch, O, name)
for name in ["simdfastpfor", "simdfastpfor-s4"]:
    T.test_mutation_fuzz_accept_reject_matches_reference(torch, R, name)
    TI.test_structural_mutations_raw(torch, O, name)
for name in TI.FP_NAMES:
    TI.test_structural_mutations_array(torch, O, name)
    TI.test_random_byte_fuzz_both_paths(torch, name)
TC.test_collisions_on_gpu(torch, O, True)
exec(TT._HEAVY.format(root={root!r}).replace('print("ok")', ''))
import runpy
sys.argv = ["team_stress.py", "20", "5"]
runpy.run_path({root!r} + "/tools/team_stress.py", run_name="__main__")
L = P._native.lib()
a = np.zeros(4, np.uint32); b = np.zeros(4, np.uint32)
assert L.izg_debug_bounds(a.ctypes.data, 0) == 0 and L.izg_debug_bounds_index(b.ctypes.data, 0) == 0
print("team decode: violations", int(a[0]), "first (kind, chunk, offset)", tuple(int(x) for x in a[1:]))
print("index kernels: violations", int(b[0]), "first (kind, chunk, offset)", tuple(int(x) for x in b[1:]))
'''
for lanes in ("0", "1000000000"):
    env = dict(os.environ, IZG_TEAM="1", IZG_SPLIT="0", IZG_INDEX_LANES_MIN=lanes)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=1800)
    print(f"== IZG_INDEX_LANES_MIN={lanes} rc={r.returncode}")
    print("\n".join(r.stdout.strip().splitlines()[-3:]))
    if r.returncode:
        print(r.stderr[-2000:])
