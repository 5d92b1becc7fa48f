"""The C++ drop-in (include/spmvkit_gpu.hpp) driven with the reference's own
TripletMatrix and generators, bitwise against the reference templates
(oracle/parity_driver.cpp, built into oracle/_ref when /root/reference was
present at build time)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "parity_driver")

pytestmark = pytest.mark.gpu


def _driver_fresh():
    """The driver compiles the header-only shim in; it is only meaningful when
    built after the last change to the headers it includes."""
    if not os.path.exists(DRIVER):
        return False
    t = os.path.getmtime(DRIVER)
    heads = [os.path.join(ROOT, "include", h) for h in ("spmvkit_gpu.hpp", "spmvk.h")]
    return all(os.path.getmtime(h) <= t for h in heads)


@pytest.mark.skipif(not _driver_fresh(), reason="oracle/_ref/parity_driver not built from this checkout")
def test_reference_inputs_through_cpp_shim(cuda):
    r = subprocess.run([DRIVER], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 6 and "FAIL" not in r.stdout
