"""bench.py's CPU-oracle baseline samples the very rows the GPU workload uses (-m "not gpu").

`bench.oracle_sample` re-creates individual rows of each config's matrices with the counter-based
generator instead of materialising them; these tests pin that re-creation to tcxgen's full-matrix
generators (the ones the GPU side uses), for every config the bench times, and smoke-run every
config's sampler for a fraction of a second."""
import numpy as np
import pytest
import torch

import bench
import tcxgen as g


def _bits(t):
    if t.dtype in (torch.float16, torch.bfloat16):
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy().view(np.uint32)
    return t.numpy()


@pytest.mark.parametrize("fmt,redraw", [("bf16", False), ("tf32", False), ("f16", False), ("f16", True), ("tf32", True)])
def test_counter_rows_match_full_matrices(fmt, redraw):
    R, n = 5, 96
    full = _bits(g.normal_matrix((R, n), fmt, 0, g.STREAM_SPVAL if redraw else g.STREAM_A, redraw_zero=redraw))
    for r in range(R):
        row = bench._counter_row_fp(0, g.STREAM_SPVAL if redraw else g.STREAM_A, r, n, fmt, redraw=redraw)
        assert np.array_equal(row, full[r]), (fmt, r)


def test_counter_rows_int8_int32_and_metadata():
    R, K = 4, 256
    assert np.array_equal(np.stack([bench._counter_row_int8(0, g.STREAM_B, r, K) for r in range(R)]),
                          g.int8_matrix((R, K), 0, g.STREAM_B).numpy())
    assert np.array_equal(np.stack([bench._counter_row_int32(0, g.STREAM_C, r, K) for r in range(R)]),
                          g.int32_matrix((R, K), 0, g.STREAM_C).numpy())
    # INT8 2:4 kept values (c4sp): [-128, 126] shifted past 0, as tcxgen.sp24_problem_i8
    v = np.stack([bench._counter_row_int32(0, g.STREAM_SPVAL, r, K // 2, -128, 126) for r in range(R)])
    vals_i8, meta = g.sp24_problem_i8(R, K, 0)
    assert np.array_equal(np.where(v >= 0, v + 1, v).astype(np.int8), vals_i8.numpy())
    # canonical 2:4 metadata rows (c5, c4sp) and 1:2 rows (c3sptf32)
    assert np.array_equal(np.stack([bench._counter_meta_row(0, r, K) for r in range(R)]), meta.numpy().view(np.uint32))
    _, meta12 = g.sp12_problem_tf32(R, K, 0)
    assert np.array_equal(np.stack([bench._counter_meta_row_sp12(0, r, K) for r in range(R)]),
                          meta12.numpy().view(np.uint32))


@pytest.mark.parametrize("cfg", ["c1", "c3", "c3tf32", "c3f16acc", "c4", "c4sp", "c3sptf32", "c5"])
def test_oracle_sample_runs(cfg):
    r = bench.oracle_sample(cfg, seconds=0.05)
    assert r["value"] > 0 and r["kind"] == "oracle" and r["cores"] >= 1 and r["unit"] in ("TFLOP/s", "TOPS", "GB/s")
