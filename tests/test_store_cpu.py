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
              "trailing_bytes", "bad_block_count", "bad_width",
              # the reference validates a half before reading the next one, and k first (from_blocks):
              # these decide on the host, before any device work
              "t_pos1_truncneg", "t_pos4_trailing", "t_k_exceeds", "k_exceeds_rows"]


@pytest.mark.parametrize("name", STRUCTURAL)
def test_structural_corruption_messages(name):
    with pytest.raises(FormatError) as exc:
        load_index(os.path.join(RSX, f"corrupt_{name}.rsx"))
    assert str(exc.value) == VERDICTS[name]


def test_k_zero_is_a_value_error():
    """column_blocks rejects k = 0 with a plain ValueError before any FormatError check, in the
    reference as here (store.py:50, indexer.py:193-199)."""
    with pytest.raises(ValueError) as exc:
        load_index(os.path.join(RSX, "corrupt_t_k_zero.rsx"))
    assert not isinstance(exc.value, FormatError)
    assert "ValueError: " + str(exc.value) == VERDICTS["t_k_zero"]


def test_header_layout():
    from paper_2411_06360_b200 import HEADER_BYTES
    assert HEADER_BYTES == 29  # <4sHBQQHI (store.py:18)
