"""Input-generator checks (synth/): the recipe in DESIGN.md §3 holds and output is thread-count independent."""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["tiny", "flickr", "yelp"])
def test_config_graph_shape(name):
    c = synth.CONFIGS[name]
    g = synth.config_graph(name)
    assert g.n_rows == c.n and g.n_cols == c.n
    assert abs(g.nnz - c.nnz) <= 0.01 * c.nnz
    deg = np.diff(g.row_ptr)
    assert deg.max() <= c.d_max() + 1
    assert deg.max() >= 0.8 * c.d_max()
    for i in range(0, g.n_rows, max(1, g.n_rows // 500)):
        cols = g.col_idx[g.row_ptr[i]:g.row_ptr[i + 1]]
        assert np.all(np.diff(cols) > 0) and (cols.size == 0 or (cols[0] >= 0 and cols[-1] < c.n))
        if cols.size:
            assert np.all(g.val[g.row_ptr[i]:g.row_ptr[i + 1]] == np.float32(1.0 / cols.size))


def test_row_block_is_bit_identical_to_full_graph():
    full = synth.power_law_graph(3000, 40000, seed=5)
    blk = synth.power_law_graph(3000, 40000, seed=5, rows=(1000, 2100))
    b0, b1 = full.row_ptr[1000], full.row_ptr[2100]
    assert np.array_equal(blk.row_ptr, full.row_ptr[1000:2101] - b0)
    assert np.array_equal(blk.col_idx, full.col_idx[b0:b1])
    assert np.array_equal(blk.val, full.val[b0:b1])


def test_thread_count_independent():
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r); import synth; "
            "g = synth.power_law_graph(20000, 300000, seed=9); x = synth.normal_f32((777, 33), 4); "
            "print(hashlib.sha256(g.row_ptr.tobytes() + g.col_idx.tobytes() + g.val.tobytes() + x.tobytes()).hexdigest())"
            % ROOT)
    outs = set()
    for nt in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=nt)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env).decode().strip())
    assert len(outs) == 1


def test_normal_moments():
    x = synth.normal_f32((1000, 256), seed=1).astype(np.float64)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01


def test_normal_row_offset_slices():
    full = synth.normal_f32((100, 7), seed=3)
    assert np.array_equal(synth.normal_f32((40, 7), seed=3, row_offset=33), full[33:73])
