"""`.rsx` parsing on the host (paper_2411_06360_b200/store.py vs reference store.py:48-101):
every structural corruption the reference rejects before touching the index arrays is
rejected here with the reference's own FormatError message (tests/golden/rsx/verdicts.json,
written by the reference's load_index).  Invariant violations need the device: see
tests/test_gpu_parity.py::test_rsx_load_golden."""

from __future__ import annotations

import json
import os

import pytest

from paper_2411_06360_b200 import FormatError, load_index

RSX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rsx")
VERDICTS = json.load(open(os.path.join(RSX, "verdicts.json")))
STRUCTURAL = ["bad_magic", "bad_version", "bad_kind", "truncated_header", "truncated_payload",
              "trailing_bytes", "bad_block_count", "bad_width"]


@pytest.mark.parametrize("name", STRUCTURAL)
def test_structural_corruption_messages(name):
    with pytest.raises(FormatError) as exc:
        load_index(os.path.join(RSX, f"corrupt_{name}.rsx"))
    assert str(exc.value) == VERDICTS[name]


def test_header_layout():
    from paper_2411_06360_b200 import HEADER_BYTES
    assert HEADER_BYTES == 29  # <4sHBQQHI (store.py:18)
