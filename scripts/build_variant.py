"""Build an A/B variant library: one CUDA source recompiled (optionally from
another path, with extra -D flags) and linked with the other cached objects.

    python scripts/build_variant.py NAME SRC_IN_CSRC [--from PATH] [-DFOO ...]

Writes paper_2504_02921_b200/_krr_NAME.so; select it with KRR_LIB=<path>.
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import build_ext as be

name, src = sys.argv[1], sys.argv[2]
rest = sys.argv[3:]
path = os.path.join(be.CSRC, src)
if rest[:1] == ["--from"]:
    path, rest = rest[1], rest[2:]
be.build()
out_dir = os.path.join(be.ROOT, "build", "variant")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"{src.replace('.cu', '')}_{name}.o")
# compile from csrc's include context even when the source comes from elsewhere
flags = list(be.FLAGS)
i = flags.index("-v")
del flags[i - 1:i + 1]                         # drop "-Xptxas -v"
subprocess.run([be.NVCC, *be.ARCH, *flags, "-I", be.CSRC, *rest,
                "-c", path, "-o", obj], check=True, capture_output=True)
objs = [os.path.join(be.BUILD, s.replace(".cu", ".o")) for s in be.SOURCES if s != src] + [obj]
lib = os.path.join(be.PKG, f"_krr_{name}.so")
subprocess.run([be.NVCC, *be.ARCH, "-shared", "-o", lib, *objs], check=True)
print(lib)
