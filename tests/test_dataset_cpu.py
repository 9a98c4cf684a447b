"""Dataset containers: the engine's FCL1 / text reader and
writer against the compiled reference's load_dataset / save_dataset
(dataset.cpp:82-111) and the golden bytes of its own test
(test_bitvec.cpp:111-136, restated). CPU only: the reader is host code."""
import os

import numpy as np
import pytest

from paper_1602_02620_b200 import fclsh as F
from tests.helpers import random_rows


def _ref(oracle_ref):
    if oracle_ref is None:
        pytest.skip("compiled reference unavailable")
    return oracle_ref


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle as O
    return O.reference() if O.reference_available() else None


def _bits(s):
    """BitVector::from_string -> row words."""
    w = np.zeros((len(s) + 63) // 64, np.uint64)
    for i, c in enumerate(s):
        if c == "1":
            w[i // 64] |= np.uint64(1) << np.uint64(i % 64)
    return w


def test_golden_container_bytes(tmp_path):
    rows = np.stack([_bits("101000000001"), _bits("010111110000")])
    path = tmp_path / "golden.bin"
    F.save_dataset(path, rows, 12)
    expected = bytes([ord("F"), ord("C"), ord("L"), ord("1"), 2, 0, 0, 0, 0, 0, 0, 0, 12, 0, 0, 0, 0, 0, 0, 0,
                      0x05, 0x08, 0xFA, 0x00])
    assert path.read_bytes() == expected
    ds = F.load_dataset(path)
    assert (ds.n, ds.dims, ds.format) == (2, 12, F.DATASET_FCL1)
    assert (ds.rows == rows).all()


@pytest.mark.parametrize("dims", [1, 7, 8, 64, 65, 130, 256])
@pytest.mark.parametrize("text", [False, True])
def test_round_trip_both_ways_with_the_reference(tmp_path, ref, dims, text):
    ref = _ref(ref)
    rng = np.random.default_rng(dims)
    rows = random_rows(rng, 20, dims)
    ours, theirs = tmp_path / "ours", tmp_path / "theirs"
    F.save_dataset(ours, rows, dims, text=text)
    ref.dataset_save(theirs, rows, dims, text=text)
    assert ours.read_bytes() == theirs.read_bytes()
    got, d = ref.dataset_load(ours)
    assert d == dims and (got == rows).all()
    ds = F.load_dataset(theirs)
    assert ds.dims == dims and ds.format == (F.DATASET_TEXT if text else F.DATASET_FCL1)
    assert (ds.rows == rows).all()


def test_large_fcl1_fast_path(tmp_path):
    rows = random_rows(np.random.default_rng(3), 5000, 512)  # d % 64 == 0: the body is the row array
    path = tmp_path / "big.bin"
    F.save_dataset(path, rows, 512)
    ds = F.load_dataset(path)
    assert ds.rows.shape == rows.shape and (ds.rows == rows).all()


def _write(path, data):
    with open(path, "wb") as f:
        f.write(data)


MALFORMED = {
    "text_width": b"0101\n011\n",
    "text_char": b"01a1\n",
    "text_empty": b"\n\n",
    "header": bytes(b"FCL1" + bytes([5, 0, 0, 0, 0, 0, 0, 0])),
    "zero_width": b"FCL1" + bytes([1] + [0] * 7) + bytes(8),
    "dirty_padding": b"FCL1" + bytes([1] + [0] * 7) + bytes([4] + [0] * 7) + bytes([0xF3]),
    "truncated_rows": b"FCL1" + bytes([3] + [0] * 7) + bytes([16] + [0] * 7) + bytes([1, 2, 3, 4, 5]),
    "trailing": b"FCL1" + bytes([1] + [0] * 7) + bytes([8] + [0] * 7) + bytes([7, 9]),
    "padding_before_truncation": b"FCL1" + bytes([4] + [0] * 7) + bytes([4] + [0] * 7) + bytes([0x03, 0x13]),
}


@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_malformed_containers_match_the_reference(tmp_path, ref, case):
    ref = _ref(ref)
    path = tmp_path / case
    _write(path, MALFORMED[case])
    with pytest.raises(F.DataError) as ours:
        F.load_dataset(path)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as theirs:
        ref.dataset_load(path)
    assert theirs.value.code == 3  # DataError
    assert f"[3] {ours.value}" == str(theirs.value)


def test_missing_file_is_a_usage_error(tmp_path):
    with pytest.raises(F.UsageError, match="cannot open"):
        F.load_dataset(tmp_path / "does_not_exist")
    with pytest.raises(F.UsageError, match="cannot open"):
        F.save_dataset(tmp_path / "no_dir" / "x.bin", np.zeros((1, 1), np.uint64), 8)


def test_text_crlf_and_blank_lines(tmp_path):
    path = tmp_path / "t.txt"
    _write(path, b"101\r\n\n011\r\n")
    ds = F.load_dataset(path)
    assert (ds.n, ds.dims, ds.format) == (2, 3, F.DATASET_TEXT)
    assert ds.rows[:, 0].tolist() == [0b101, 0b110]
    os.remove(path)
