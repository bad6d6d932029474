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
