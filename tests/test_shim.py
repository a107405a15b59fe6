"""The INTEGRATION.md shim (integration/placers_b200.cpp): the reference's
own place_mtopo / place_metf / place_msct signatures forwarded to the C ABI,
compiled against /root/reference/proj/include by oracle/Makefile (target
`shim`) into oracle/_ref/shim_driver, which runs it next to the unmodified
reference placer (renamed ref_place_*) on reference-typed inputs."""
import json
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "oracle", "_ref", "shim_driver")

needs_driver = pytest.mark.skipif(not os.path.exists(DRIVER), reason="shim driver not built (no reference sources)")


def _run():
    r = subprocess.run([DRIVER], capture_output=True, text=True, timeout=900)
    return r.returncode, json.loads(r.stdout.strip().splitlines()[-1])


@needs_driver
def test_shim_fails_loudly_without_gpu():
    """No CUDA device: every shim call raises the engine's 'no CPU fallback'
    error (never a silent CPU placement)."""
    import paper_2301_08695_b200 as bx
    if bx.device_count() > 0:
        pytest.skip("a GPU is present")
    rc, s = _run()
    assert rc == 1 and s["mismatches"] == s["cases"] > 0
    assert "no CPU fallback" in s["first_mismatch"]


@pytest.mark.gpu
@needs_driver
def test_shim_matches_reference_placer():
    """Every case: the same Placement + PlacerStats, or the same exception
    kind and what() text, as the reference placer."""
    rc, s = _run()
    assert rc == 0 and s["mismatches"] == 0, s
    assert s["cases"] >= 800 and s["reference_errors"] > 0
