"""Shared pytest wiring: the ``gpu`` marker and golden-file loaders."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built liblms.so")
    _install_pool_if_gpu()


_POOL = {}


def _install_pool_if_gpu():
    """On a GPU box, route every torch CUDA allocation of the test session through
    liblms's pool (must happen before the first CUDA allocation)."""
    if os.environ.get("LMS_TEST_NO_POOL"):
        return
    try:
        import torch
    except Exception:
        return
    if not torch.cuda.is_available():
        return
    from paper_1807_02037_b200 import runtime as rt
    ctx = rt.Context(device=0, device_reserve=24 << 30, host_chunk=1 << 30, timing=True)
    rt.install_allocator(ctx)
    _POOL["ctx"] = ctx


@pytest.fixture(scope="session")
def lms_ctx():
    """The session's liblms context (its pool backs every torch CUDA tensor)."""
    if "ctx" not in _POOL:
        pytest.skip("no CUDA device / liblms pool")
    return _POOL["ctx"]


def load_golden(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def rewrite_cases():
    return load_golden("rewrite_cases.json.gz")


@pytest.fixture(scope="session")
def ctrl_cases():
    return load_golden("ctrl_queries.json.gz")


@pytest.fixture(scope="session")
def interp_cases():
    return load_golden("interp_cases.json.gz")


@pytest.fixture(scope="session")
def sim_cases():
    return load_golden("sim_cases.json.gz")
