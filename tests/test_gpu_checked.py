"""The checked diagnosis build: the library compiled with -DFIKIT_CHECKS, whose device-side
invariant checks (FK_CHECK in csrc/: tile positions and TMA sources in range, hot-slot indices
below the admitted count and their rows below the capacity, the tile-group scatter in range, every
pick of an alive request that fits, finalize ranks below K) print and trap when violated.  The
small parity cases -- the selection scripts/sanitize.sh ran under compute-sanitizer, which the GPU
pool no longer offers -- rerun on it in a subprocess, each still compared with the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEL = ("toy_end_to_end or (measure_random and not 300000 and not 70000) or identify_random or invalid_record or "
       "capacity_and_empty or test_halo or test_random_replay or fill_batch or predict_parity or empty_inputs or "
       "lookup_parity or merge_one_gpu or stream_singletons or stream_limits or over_limit or sorted_pool_beyond or "
       "zero_durations or zipf_small_full or resnet_full")


def test_parity_cases_on_the_checked_build():
    from conftest import cuda_ok

    if not cuda_ok():
        pytest.skip("no CUDA device")
    from paper_2311_10359_b200 import _build

    lib = _build.build(defines=("FIKIT_CHECKS",), out=os.path.join(ROOT, "build", "checked", "libfikit.so"))
    env = dict(os.environ, FIKIT_DIAG_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "tests/test_gpu_edges.py", "-m", "gpu",
                        "-q", "-x", "-p", "no:cacheprovider", "-k", SEL], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "FIKIT_CHECK failed" not in r.stdout + r.stderr, tail
    assert " passed" in r.stdout, tail
