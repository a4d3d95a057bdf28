"""The C++ drop-in (include/gsim_gpu.hpp) against the reference in one binary, on the GPU.

oracle/_ref/drop_in_check is built by `make -C oracle drop_in` (__graft_entry__.build()) where the
reference sources exist; it links the unmodified reference library as the checker and
libgsim_gpu.so through gsim::gpu::render / project / rasterize / transform_primitives with the
reference's own types, and exits non-zero on any parity failure.
"""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "drop_in_check"


def test_cpp_drop_in_matches_reference():
    if not BIN.exists():
        pytest.skip("drop_in_check not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "DROP-IN OK" in res.stdout
