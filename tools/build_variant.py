"""Build an A/B variant of libpfgpu.so: recompile ONE translation unit with
extra nvcc flags and link it with the other objects of the in-tree build.

usage: python tools/build_variant.py <tu.cu> <tag> [-DFOO=1 ...]
  -> paper_2304_07338_b200/libpfgpu_<tag>.so (load with PF_LIBPFGPU=<path>)
Tooling, not product.
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2304_07338_b200 import build as b  # noqa: E402

tu, tag, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
obj = b.BUILD / f"{Path(tu).stem}_{tag}.o"
cmd = [b._nvcc(), *b.ARCH, *b.COMMON, *b.SOURCES[tu], *extra, "-I", str(b.INCLUDE), "-c", str(b.CSRC / tu),
       "-o", str(obj)]
subprocess.run(cmd, check=True)
objs = [str(obj) if o.name == tu.replace(".cu", ".o") else str(o)
        for o in (b.BUILD / s.replace(".cu", ".o") for s in b.SOURCES)]
out = b.HERE / f"libpfgpu_{tag}.so"
subprocess.run([b._nvcc(), *b.ARCH, "-shared", "-cudart", "static", "-o", str(out), *objs], check=True)
print(out)
