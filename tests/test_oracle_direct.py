"""Pins for oracle.direct (the float64 direct correlation, Eq. (2)).

Pinned against: hand sums from the paper/SPEC examples, a textbook library
routine (torch float64 convNd on CPU -- independent of both oracle and the
CUDA path), a second implementation (pure-Python brute force), linearity and
the output-extent contract.
"""
import numpy as np
import pytest
import torch

from oracle import direct


def test_worked_1d_example():
    # (1,2,3,4) correlated with (1,1,1) = (6, 9)
    x = np.array([[[1, 2, 3, 4]]], np.float32)
    g = np.array([[[1, 1, 1]]], np.float32)
    y = direct.direct_conv_f64(x, g, 0)
    assert y.tolist() == [[[6.0, 9.0]]]
    assert direct.direct_conv_py(x, g, 0).tolist() == [[[6.0, 9.0]]]


def test_not_flipped():
    # cross-correlation, no kernel flip (reading #1): g=(1,0,0) picks d[o]
    x = np.array([[[5, 7, 11, 13]]], np.float32)
    g = np.array([[[1, 0, 0]]], np.float32)
    assert direct.direct_conv_f64(x, g, 0).tolist() == [[[5.0, 7.0]]]


def test_ones_2d():
    # 3x3 ones (*) 2x2 ones = 2x2 of 4s
    y = direct.direct_conv_f64(np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 2, 2), np.float32), 0)
    assert np.array_equal(y, np.full((1, 1, 2, 2), 4.0))


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_delta_kernel_identity(N):
    rng = np.random.default_rng(N)
    x = rng.standard_normal((2, 1) + (4,) * N).astype(np.float32)
    g = np.zeros((1, 1) + (3,) * N, np.float32)
    g[(0, 0) + (1,) * N] = 1.0            # centred delta with pad 1 -> identity
    y = direct.direct_conv_f64(x, g, 1)
    assert np.array_equal(y, x.astype(np.float64))


def test_delta_two_channels_sum():
    # g^(1,1) = g^(1,2) = delta -> channel sum
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 2, 5, 6)).astype(np.float32)
    g = np.ones((1, 2, 1, 1), np.float32)
    y = direct.direct_conv_f64(x, g, 0)
    assert np.array_equal(y[0, 0], x[0, 0].astype(np.float64) + x[0, 1].astype(np.float64))


@pytest.mark.parametrize("in_dims,r,pad", [((7,), 3, 0), ((8, 5), 3, 1), ((4, 6, 5), 3, 2), ((9, 9), 4, 1)])
def test_output_extent(in_dims, r, pad):
    x = np.zeros((1, 1) + in_dims, np.float32)
    g = np.zeros((1, 1) + (r,) * len(in_dims), np.float32)
    y = direct.direct_conv_f64(x, g, pad)
    assert y.shape[2:] == tuple(i + 2 * pad - r + 1 for i in in_dims)


def test_kernel_larger_than_padded_input_rejected():
    with pytest.raises(ValueError):
        direct.direct_conv_f64(np.zeros((1, 1, 2, 2), np.float32), np.zeros((1, 1, 5, 5), np.float32), 0)


def test_linearity():
    rng = np.random.default_rng(2)
    a = rng.integers(-8, 8, (2, 3, 6, 7)).astype(np.float32)
    b = rng.integers(-8, 8, (2, 3, 6, 7)).astype(np.float32)
    g = rng.integers(-4, 4, (4, 3, 3, 3)).astype(np.float32)
    ya = direct.direct_conv_f64(a, g, 1)
    yb = direct.direct_conv_f64(b, g, 1)
    yab = direct.direct_conv_f64(2 * a - 3 * b, g, 1)
    assert np.array_equal(yab, 2 * ya - 3 * yb)       # small integers: exact in f64


@pytest.mark.parametrize("N,shape,r,pad", [
    (1, (3, 4, 11), 3, 1),
    (2, (2, 3, 9, 7), 3, 1),
    (2, (2, 2, 8, 8), 4, 0),
    (3, (2, 3, 5, 6, 7), 3, 1),
    (3, (1, 2, 4, 4, 5), 3, 2),
])
def test_vs_torch_conv_f64(N, shape, r, pad):
    rng = np.random.default_rng(N * 10 + r)
    x = rng.standard_normal(shape).astype(np.float32)
    K = 5
    g = rng.standard_normal((K, shape[1]) + (r,) * N).astype(np.float32)
    y = direct.direct_conv_f64(x, g, pad)
    conv = {1: torch.nn.functional.conv1d, 2: torch.nn.functional.conv2d,
            3: torch.nn.functional.conv3d}[N]
    ref = conv(torch.from_numpy(x).double(), torch.from_numpy(g).double(), padding=pad).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_vs_torch_4d_as_sum_of_conv3d():
    # N=4: sum over the first kernel axis of conv3d on shifted input slices
    rng = np.random.default_rng(44)
    B, C, K, r, pad = 2, 3, 2, 3, 1
    x = rng.standard_normal((B, C, 4, 5, 4, 6)).astype(np.float32)
    g = rng.standard_normal((K, C) + (r,) * 4).astype(np.float32)
    y = direct.direct_conv_f64(x, g, pad)
    xt = torch.nn.functional.pad(torch.from_numpy(x).double(), (0, 0, 0, 0, 0, 0, pad, pad))
    gt = torch.from_numpy(g).double()
    out1 = x.shape[2] + 2 * pad - r + 1
    ref = torch.zeros(y.shape, dtype=torch.float64)
    for o in range(out1):
        for p in range(r):
            ref[:, :, o] += torch.nn.functional.conv3d(xt[:, :, o + p], gt[:, :, p], padding=pad)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_c_vs_python_bruteforce(N):
    rng = np.random.default_rng(100 + N)
    shape = (2, 2) + (3,) * (N - 1) + (4,)
    x = rng.integers(-5, 6, shape).astype(np.float32)
    g = rng.integers(-3, 4, (2, 2) + (2,) * N).astype(np.float32)
    y = direct.direct_conv_f64(x, g, 1)
    yp = direct.direct_conv_py(x, g, 1).astype(np.float64)
    assert np.array_equal(y, yp)


def test_sampled_equals_full():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((2, 3, 6, 5, 7)).astype(np.float32)
    g = rng.standard_normal((4, 3, 3, 3, 3)).astype(np.float32)
    y = direct.direct_conv_f64(x, g, 1)
    idx = rng.integers(0, y.size, 50)
    v = direct.direct_conv_at(x, g, 1, idx)
    assert np.array_equal(v, y.reshape(-1)[idx])
