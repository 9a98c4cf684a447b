"""write_metrics (bench.cpp:160-170): the engine's CSV is byte-identical to
the reference's own writer (oracle/_ref/ref_write_metrics) on the same rows."""
import io
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_1602_02620_b200.experiment import MetricsRow, write_metrics

REF_BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "ref_write_metrics")


def test_csv_is_byte_identical_to_the_reference(tmp_path):
    if not os.path.exists(REF_BIN):
        pytest.skip("compiled reference unavailable")
    rng = np.random.default_rng(4)
    rows = [MetricsRow(0, "fclsh", 8, 102.5, 1.0, 1.0, 1.0, 1.0, 1.0, 1.1074999999999999, 0.1, 3.0),
            MetricsRow(1, "fclsh", 8, 511.0 / 3, 2.0 / 3, 0.0, 0.0, 1.0, 1.0, 0.0, 1e-9, 12345678.9)]
    for q in range(2, 40):
        v = rng.random(9) * 10.0 ** rng.integers(-6, 9, 9)
        rows.append(MetricsRow(q, "fclsh", 8, *[float(x) for x in v]))
    blob = struct.pack("<Q", len(rows)) + b"".join(
        struct.pack("<12d", r.query_id, r.radius, r.collisions, r.candidates, r.found, r.true_near, r.precision,
                    r.recall, r.time_s1_us, r.time_s2_us, r.time_s3_us, 0.0) for r in rows)
    path = tmp_path / "rows.bin"
    path.write_bytes(blob)
    want = subprocess.run([REF_BIN, str(path), "fclsh"], capture_output=True, check=True).stdout.decode()
    out = io.StringIO()
    write_metrics(rows, out)
    assert out.getvalue() == want
