"""The C++ drop-in (include/bsccs_b200_solver.hpp) used at a reference call
site: bsccs::fit vs bsccs_b200::fit on the reference's own types, plus the
status -> reference-exception mapping.  The binary is built where the
reference headers exist (build.py build_cpp_tests) and run on the GPU."""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parent / "cpp" / "_bin" / "test_shim"


def test_shim_header_is_self_contained_c_abi():
    hdr = (Path(__file__).resolve().parents[1] / "include" / "bsccs_b200_solver.hpp").read_text()
    assert '#include "bsccs_b200.h"' in hdr and "solver.hpp:206-210" in hdr


@pytest.mark.gpu
def test_cpp_shim_matches_reference_fit():
    if not EXE.exists():
        pytest.skip("test_shim not built (needs the reference headers at build time)")
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "-> OK" in out.stdout
