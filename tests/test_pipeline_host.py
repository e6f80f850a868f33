"""Chunk schedules of the host-memory pipeline (pipeline.py), no GPU."""

import pytest

from paper_2509_07120_b200.pipeline import ramp_chunks


@pytest.mark.parametrize("heads", list(range(1, 40)))
def test_ramp_chunks_cover_heads(heads):
    sizes = ramp_chunks(heads)
    assert sum(sizes) == heads and all(1 <= s <= 4 for s in sizes)
    assert sizes[0] == 1 and sizes[-1] == 1


def test_ramp_chunks_bench_shape():
    assert ramp_chunks(16) == [1, 3, 4, 4, 3, 1]
