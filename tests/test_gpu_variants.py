"""The non-default decode variants (multi-head CTAs, alternate grid order and
split sizes) must be exactly as correct as the default: rerun the decode
parity tests in subprocesses with the tuning knobs set."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env", [
    {"JENGA_DECODE_HEADS_PER_CTA": "2"},
    {"JENGA_DECODE_HEADS_PER_CTA": "4"},
    {"JENGA_DECODE_GRID_ORDER": "1", "JENGA_DECODE_TILES_PER_SPLIT": "8"},
])
def test_decode_variants_parity(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", str(ROOT / "tests" / "test_gpu_parity.py"),
                        "-k", "gemma or decode_shapes or cross or toy"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_prefill_mma_sync_variant_parity():
    """JENGA_PREFILL_TC5=0 selects the mma.sync prefill kernel (prefill.cu)."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", str(ROOT / "tests" / "test_gpu_prefill.py")],
                       env=dict(os.environ, JENGA_PREFILL_TC5="0"), capture_output=True, text=True, timeout=900,
                       cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
