"""Developer A/B builds: compile the library with extra -D flags into
paper_1209_2137_b200/_lib/variants/<name>.so (load with IZG_LIB_PATH=...).

    python tools/build_variant.py NAME -DIZG_FLAT_PATCH=0 ...
"""
import os, shutil, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_2137_b200 import build as B

name, flags = sys.argv[1], sys.argv[2:]
os.environ["IZG_NVCC_EXTRA"] = " ".join(flags)
B.LIB = os.path.join(B.LIBDIR, "variants", name + ".so")
os.makedirs(os.path.dirname(B.LIB), exist_ok=True)
B.OBJDIR = B.LIB + ".obj"
print(B.build(force=True))
