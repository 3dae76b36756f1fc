"""The driver's round-end entry point: ``__graft_entry__.smoke()`` runs the
tensor-core, tile and warp forward paths on cuda:0 against the oracle."""

from __future__ import annotations

import os
import sys

import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu


def test_smoke_entry_point():
    if not cuda_ok():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import __graft_entry__

    __graft_entry__.smoke()
