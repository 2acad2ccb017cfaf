"""The device expf/tanhf/expm1f ports (csrc/glibc_mathf.h) against the host
libm the reference links, on a strided sample of all 2^32 float inputs (the
full exhaustive sweep is `build/libm_exhaustive 1`, ~30 s on 8 cores)."""
import os
import subprocess

from conftest import ROOT


def test_libm_port_bit_exact_sampled():
    exe = os.path.join(ROOT, "build", "libm_exhaustive")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-pthread", "-o", exe,
                    os.path.join(ROOT, "tests", "native", "libm_exhaustive.c"), "-lm"], check=True)
    out = subprocess.run([exe, "61"], capture_output=True, text=True)
    lines = dict((l.split()[0], l.split()[1:]) for l in out.stdout.strip().splitlines())
    for fn in ("expf", "tanhf", "expm1f"):
        checked, bad, _ = lines[fn]
        assert int(checked) > 70_000_000 and int(bad) == 0, (fn, lines[fn])
