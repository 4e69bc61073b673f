"""The committed golden fixtures are exactly what the reference produces:
regenerate them with tests/golden/make_golden.py from the real reference
(only where /root/reference is importable, i.e. the build container) into a
scratch tree and compare byte for byte / array for array."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path(os.environ.get("VOXGRID_REF", "/root/reference/pkg/src"))


@pytest.mark.skipif(not (REF / "voxgrid").is_dir(), reason="reference package not present")
def test_golden_fixtures_regenerate_identically(tmp_path):
    repo = tmp_path / "repo"
    (repo / "tests" / "golden").mkdir(parents=True)
    shutil.copy(ROOT / "tests" / "golden" / "make_golden.py", repo / "tests" / "golden")
    for name in ("paper_2211_08506_b200", "oracle"):
        (repo / name).symlink_to(ROOT / name)
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    res = subprocess.run([sys.executable, "tests/golden/make_golden.py"], cwd=repo, env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    a, b = ROOT / "tests" / "golden", repo / "tests" / "golden"
    for f in ("configs.json", "io.json", "reversal.json"):
        assert (a / f).read_text() == (b / f).read_text(), f
    for f in ("erf.npz", "tables.npz", "grids.npz"):
        x, y = np.load(a / f), np.load(b / f)
        assert sorted(x.files) == sorted(y.files), f
        for k in x.files:
            assert np.array_equal(x[k], y[k]), (f, k)
