"""Seeded input generators (inputs/): shape and reproducibility checks."""
import numpy as np
import pytest

import inputs


def test_draw_is_splitmix64():
    # first outputs of SplitMix64 seeded with 0 (Steele, Lea, Flood 2014 reference values)
    assert inputs.draw(0, 0) == 0xE220A8397B1DCDAF
    assert inputs.draw(0, 1) == 0x6E789E6AA1B965F4


def test_er_exact_edges_no_loops_no_duplicates():
    src, dst = inputs.er(1000, 5000, 13111)
    assert len(src) == 5000 and (src != dst).all()
    key = np.minimum(src, dst).astype(np.int64) << 32 | np.maximum(src, dst)
    assert len(np.unique(key)) == 5000
    assert src.min() >= 0 and max(src.max(), dst.max()) < 1000
    s2, d2 = inputs.er(1000, 5000, 13111)
    assert np.array_equal(src, s2) and np.array_equal(dst, d2)


def test_grid_counts():
    src, dst = inputs.grid(2048)
    assert len(src) == 8_384_512
    assert ((dst - src == 1) | (dst - src == 2048)).all()


def test_rmat_range_and_skew():
    src, dst = inputs.rmat(12, 16 << 12, 0.57, 0.19, 0.19, 5)
    assert src.max() < 4096 and dst.max() < 4096 and src.min() >= 0
    # P(bit = 0) = a + b = 0.76 per level: vertex 0 is by far the most frequent source
    assert np.bincount(src).argmax() == 0


def test_chung_lu_heavy_head():
    src, dst = inputs.chung_lu(10000, 2.1, 200000, 3)
    deg = np.bincount(np.concatenate([src, dst]), minlength=10000)
    assert deg[0] == deg.max() and deg[0] > 50 * np.median(deg[deg > 0])


def test_weights():
    w = inputs.uniform_weights(100000, 7)
    assert w.dtype == np.float32 and w.min() >= 1.0 and w.max() < 10.0
    e = inputs.exp_weights(100000, 7)
    assert e.min() >= 0 and abs(e.mean() - 1.0) < 0.02


def test_terminals_distinct():
    t = inputs.terminals(2048 * 2048, 25, 9)
    assert len(set(t.tolist())) == 25


@pytest.mark.gpu
def test_device_twin_matches_host():
    import torch
    n = 1 << 14
    src_h, dst_h = inputs.rmat(14, n, 0.57, 0.19, 0.19, 77)
    s = torch.empty(n, dtype=torch.int32, device="cuda")
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    inputs.rmat_device(14, n, 0.57, 0.19, 0.19, 77, s.data_ptr(), d.data_ptr(), stream)
    w = torch.empty(n, dtype=torch.float32, device="cuda")
    inputs.uniform_weights_device(n, 78, w.data_ptr(), stream)
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), src_h) and np.array_equal(d.cpu().numpy(), dst_h)
    assert np.array_equal(w.cpu().numpy(), inputs.uniform_weights(n, 78))
