"""GPU: the reference's dense kernel table (tensor::gemm / hadamard / activate / scale_rows,
tensor/kernels.hpp:26-39, ops.cpp:24-95) through the C ABI (nsdf_cuda_tensor_*), bit for bit
against the reference library's AVX2 backend (oracle/_ref) on random and awkward shapes:
panel and column-tail widths, k = 0, with and without bias, f32 and f64, sine arguments over
many quadrants and its derivative."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(oracle_built):
    from oracle import refshim
    refshim.set_backend("avx2")
    return refshim


@pytest.fixture(scope="module")
def dev():
    from paper_2201_09147_b200.engine import Context
    c = Context(0, "fp32")
    yield c
    c.close()


SHAPES = [(1, 1, 1), (2, 1, 2), (5, 37, 13), (4, 16, 7), (7, 33, 64), (64, 300, 64), (256, 1024, 256), (3, 17, 0)]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_gemm_bitwise(ref, dev, dtype, m, n, k):
    rng = np.random.default_rng(m * 1000 + n * 10 + k)
    a = rng.normal(size=(m, k)).astype(dtype)
    b = rng.normal(size=(k, n)).astype(dtype)
    bias = rng.normal(size=m).astype(dtype)
    for bb in (None, bias):
        got = dev.tensor_gemm(a, b, bb)
        want = ref.tensor_op(0, a, b, bb, m=m, n=n, k=k)
        assert got.dtype == dtype and np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_gemm_hand_example(dev):
    # test_tensor.cpp:41-46: [[1,2],[3,4]] . [1,1]^T + 10 = [13, 17]
    c = dev.tensor_gemm(np.array([[1, 2], [3, 4]], np.float32), np.ones((2, 1), np.float32),
                        np.array([10, 10], np.float32))
    assert c.reshape(-1).tolist() == [13.0, 17.0]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_elementwise_bitwise(ref, dev, dtype):
    rng = np.random.default_rng(7)
    m, n = 37, 129
    a = rng.normal(size=(m, n)).astype(dtype)
    b = rng.normal(size=(m, n)).astype(dtype)
    col = rng.normal(size=(m, 1)).astype(dtype)
    assert np.array_equal(dev.tensor_hadamard(a, b), ref.tensor_op(1, a, b, m=m, n=n))
    assert np.array_equal(dev.tensor_scale_rows(col, b), ref.tensor_op(3, col, b, m=m, n=n))
    x = (rng.uniform(-3, 3, size=(m, n)) * rng.choice([1, 10, 100], size=(m, n))).astype(dtype)
    for omega in (1.0, 30.0):
        for deriv in (False, True):
            got = dev.tensor_sine(x, omega, deriv)
            want = ref.tensor_op(2, x, m=m, n=n, omega=omega, derivative=deriv)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_sine_at_zero(dev):
    # test_tensor.cpp:153-155: sine(0) = 0, derivative omega
    z = np.zeros((1, 4), np.float32)
    assert np.all(dev.tensor_sine(z, 1.0) == 0.0) and np.all(dev.tensor_sine(z, 1.0, True) == 1.0)


def test_contract_errors(dev):
    from paper_2201_09147_b200.abi import NsdfError
    with pytest.raises(NsdfError):
        dev.tensor_gemm(np.zeros((2, 2), np.int32), np.zeros((2, 2), np.int32))
