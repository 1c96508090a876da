"""The C ABI from a plain C++ host (no Python on the path, no reference
headers): tests/cpp/capi_frame.cpp is compiled against include/pf_gpu.h and
libpfgpu.so and runs neural / path-traced / photon-map renders, photon
tracing, the training loop and an error path on the GPU."""
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_c_abi_host_program(tmp_path):
    from paper_2304_07338_b200 import _lib
    if not shutil.which("g++"):
        pytest.skip("g++ not present")
    libdir = _lib.LIB_PATH.parent
    exe = tmp_path / "capi_frame"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "capi_frame.cpp"),
                    "-o", str(exe), f"-L{libdir}", "-lpfgpu", f"-Wl,-rpath,{libdir}"], check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi ok" in r.stdout and "finite=1" in r.stdout
