"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run only on a B200
(`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLD = os.path.join(REPO, "tests", "golden")
#: the reference package installed by oracle/build_ref.py (git-ignored, shipped
#: to the GPU box): the drop-in tests run its own driver and front end
REF_INSTALL = os.path.join(REPO, "oracle", "_ref")
if os.path.isdir(REF_INSTALL) and REF_INSTALL not in sys.path:
    sys.path.append(REF_INSTALL)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsylvadi_b200.so")
    config.addinivalue_line("markers", "slow: long-running (minutes)")


@pytest.fixture
def rng():
    # same seed as the reference's conftest (pkg/tests/conftest.py:106-108)
    return np.random.default_rng(20260826)


def read_steps_csv(path):
    """Per-step records of a golden CSV as a list of dicts."""
    with open(path) as fh:
        head = fh.readline().strip().split(",")
        rows = []
        for line in fh:
            vals = line.strip().split(",")
            if len(vals) != len(head):
                continue
            rec = {}
            for k, v in zip(head, vals):
                rec[k] = int(v) if k in ("step", "inner_it_A", "inner_it_B") else float(v)
            rows.append(rec)
    return rows
