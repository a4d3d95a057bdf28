"""C-ABI boundary checks that need no GPU: the library builds, loads and exports every entry
point include/gsim_gpu.h declares; the structs match the reference layouts; there is no silent
CPU fallback when no device is present."""
from __future__ import annotations

import ctypes as C
import subprocess

import numpy as np
import pytest

from paper_2507_21981_b200 import abi


@pytest.fixture(scope="module")
def lib():
    if not abi.LIB_PATH.exists():
        from paper_2507_21981_b200.build import build
        build()
    return abi.load_library()


def test_exports_every_header_symbol(lib):
    declared = abi.header_symbols()
    assert len(declared) >= 19
    out = subprocess.run(["nm", "-D", "--defined-only", str(abi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for name in declared:
        assert hasattr(lib, name)
    assert {name for name, _, _ in abi.SIGNATURES} == set(declared)


def test_struct_layouts():
    # ProjectedSplat (raster.hpp:20-29) is 120 bytes with the same field offsets
    assert C.sizeof(abi.gsim_projected_splat) == 120
    assert abi.gsim_projected_splat.prim_index.offset == 112
    assert C.sizeof(abi.gsim_rigid) == 56
    assert C.sizeof(abi.gsim_camera) == 4 * 8 + 8 + 56 + 16 + 8
    assert C.sizeof(abi.gsim_node) == 16 + 56 + 8
    assert abi.SPLAT_DTYPE.itemsize == 120


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_string(lib):
    assert b"sm_100a" in lib.gsim_gpu_version()


def test_no_cpu_fallback_without_device(lib):
    """Creating a context either yields a real CUDA context or fails loudly (status 1/2)."""
    p = C.c_void_p()
    st = lib.gsim_gpu_context_create(0, C.byref(p))
    if st == abi.GSIM_OK:
        lib.gsim_gpu_context_destroy(p)
    else:
        assert st in (abi.GSIM_ERR_IO, abi.GSIM_ERR_VALIDATION)
        assert lib.gsim_gpu_last_error(None)


def test_null_context_is_validation_error(lib):
    assert lib.gsim_gpu_synchronize(None) == abi.GSIM_ERR_VALIDATION


def test_field_view_strides_cover_aos_and_soa():
    """The C view accepts the reference's AoS GaussianPrimitive (59 doubles) and SoA numpy."""
    from paper_2507_21981_b200.api import GaussianField
    n = 5
    aos = np.arange(n * 59, dtype=np.float64).reshape(n, 59)
    f = GaussianField(aos[:, 0:3], aos[:, 3:6], aos[:, 6:10], aos[:, 10], aos[:, 11:59], 3)
    v = f.view()
    assert v.count == n and v.means_stride == 3 and v.sh_stride == 48
    assert v.means[3 * 2 + 1] == aos[2, 1]
    assert v.sh[48 * 4 + 47] == aos[4, 58]


def test_hash_target_matches_reference_hash(lib, oracle):
    """gsim_gpu_hash_target (host FNV-1a) equals hash.hpp:36-41 as restated by the oracle (pinned
    to the reference's own image hashes in test_oracle_pin.py), chained seeds included."""
    from paper_2507_21981_b200.api import RenderTarget
    rng = np.random.default_rng(5)
    t = RenderTarget(rng.random((7, 9, 3), dtype=np.float32), rng.random((7, 9), dtype=np.float32),
                     rng.random((7, 9), dtype=np.float32))
    assert t.hash() == oracle.hash_target(t)
    assert t.hash(12345) == oracle.hash_target(t, 12345)
    bad = RenderTarget(t.rgb.astype(np.float64), t.depth, t.accum_alpha)
    from paper_2507_21981_b200 import ValidationError
    with pytest.raises(ValidationError):
        bad.hash()


def test_bench_refuses_mismatched_world_size():
    """bench.py --gpus N under a launcher whose WORLD_SIZE differs exits non-zero (it never
    silently reports fewer GPUs than asked)."""
    import json
    import os
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2
    assert "WORLD_SIZE" in json.loads(r.stdout.strip().splitlines()[-1])["error"]


def test_bench_reference_arm_self_launches_two_ranks():
    """--gpus 2 outside torchrun re-launches under torch.distributed.run; in the reference arm
    rank 0 alone times the reference's CPU renderer (oracle/_ref) and prints one JSON line with
    impl = reference, the other rank exits 0 without work."""
    import json
    import os
    import sys
    from pathlib import Path
    from oracle.oracle import REF_LIB
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built")
    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "cfg0", "--steps", "1", "--warmup", "3"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and len(d["first_frame_hash"]) == 16
    assert d["e2e"]["h2d_bytes_per_step"] == 0
