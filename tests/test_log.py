"""The PARITY tracers' binary64 log (paper_2304_07338_b200/csrc/pf_log.h),
compiled for the host from the same source (identical operations: explicit
fma, no contraction), against glibc's log -- the reference's std::log
(proj/src/volume.cpp:217, 247).  CPU only.

Tolerance: at most 1 ulp from glibc anywhere; over 2e7 tracer-domain inputs
(1 - k 2^-53) <= 1e-3 differ at all (glibc itself is not correctly rounded in
~9e-4 of them; pf_log is nearer to correct rounding than glibc), and log(1)
is +0 exactly.
"""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_pf_log_matches_glibc(tmp_path):
    exe = tmp_path / "log_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17",
                    "-I", str(ROOT / "paper_2304_07338_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "log_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True, check=True).stdout.split()
    n, diff, diff_wide, worst, one = map(int, out)
    print(f"{diff} of {n} differ, {diff_wide} of {n // 10} wide-range, worst {worst} ulp")
    assert one == 1
    assert worst <= 1
    assert diff <= 1e-3 * n
    assert diff_wide <= 1e-3 * (n // 10)
