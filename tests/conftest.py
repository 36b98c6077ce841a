"""Shared pytest setup: the `gpu` marker, repo on sys.path, fixture loaders."""

from __future__ import annotations

import gzip
import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def load_golden(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_schedules():
    return load_golden("schedules.json.gz")


@pytest.fixture(scope="session")
def golden_decompositions():
    return load_golden("decompositions.json.gz")


@pytest.fixture(scope="session")
def golden_generators():
    return load_golden("generators.json.gz")


def reference_available() -> bool:
    return os.path.isdir("/root/reference/pkg/src/tiersched")


def import_reference():
    """Import tiersched from the read-only reference tree (CPU tests only)."""
    sys.dont_write_bytecode = True
    p = "/root/reference/pkg/src"
    if p not in sys.path:
        sys.path.insert(0, p)
    import tiersched

    return tiersched
