"""SIREN training on the GPU vs the reference trainer, bit for bit:
training-set sampling, backprop_sine_mlp gradients, and whole fit_mlp runs (shuffles,
minibatch chunking, momentum, warmup, checkpoint / rollback / plateau schedule, validation)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TORUS = "torus:R=0.6,r=0.3"


def _u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def ref(oracle_built):
    from oracle import refshim
    refshim.set_backend("avx2")
    return refshim


def test_sample_training_set(ref):
    from paper_2201_09147_b200 import train
    a = train.sample_training_set(TORUS, 3000, 2000, 0.01, 500, seed=4)
    b = ref.sample_training_set(TORUS, 3000, 2000, 0.01, 500, seed=4)
    for x, y in zip(a, b):
        assert np.array_equal(_u64(x), _u64(y))


@pytest.mark.parametrize("arch,k", [("16x1", 1), ("64x1", 777), ("128x2", 4096), ("64x2", 5000), ("256x3", 300)])
def test_backprop_bitexact(ref, arch, k):
    from paper_2201_09147_b200 import train
    rng = np.random.default_rng(k)
    pts = rng.uniform(-1, 1, (3, k))
    tg = np.linalg.norm(pts, axis=0) - 0.7
    pa, ga, la = train.backprop(arch, pts, tg, seed=11)
    pb, gb, lb = ref.backprop(arch, pts, tg, seed=11)
    assert np.array_equal(_u64(pa), _u64(pb))  # random_init matches
    assert np.array_equal(_u64(ga), _u64(gb))
    assert _u64([la]) == _u64([lb])


def test_backprop_4d(ref):
    from paper_2201_09147_b200 import train
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (4, 900))
    tg = np.linalg.norm(pts[:3], axis=0) - 0.5 * pts[3]
    _, ga, la = train.backprop("64x1", pts, tg, seed=2)
    _, gb, lb = ref.backprop("64x1", pts, tg, seed=2)
    assert np.array_equal(_u64(ga), _u64(gb)) and _u64([la]) == _u64([lb])


@pytest.mark.parametrize("arch,epochs,batch,lr", [("32x1", 12, 1000, 0.3), ("64x2", 8, 0, 0.1), ("32x1", 30, 700, 50.0)])
def test_fit_mlp_bitexact(ref, arch, epochs, batch, lr):
    """Whole training runs; the last case diverges on purpose (rollback + halvings)."""
    from paper_2201_09147_b200 import train
    from paper_2201_09147_b200.abi import TrainConfigC
    pts, tg, vp, vt = ref.sample_training_set(TORUS, 4000, 3000, 0.01, 800, seed=9)
    cfg = TrainConfigC(epochs=epochs, batch_size=batch, learning_rate=lr, warmup_epochs=3, plateau_patience=4,
                       plateau_threshold=0.05)
    pa, la, ra = train.fit_mlp(arch, pts, tg, vp, vt, cfg, seed=5)
    pb, lb, rb = ref.fit_mlp(arch, pts, tg, vp, vt, cfg, seed=5)
    assert np.array_equal(_u64(la), _u64(lb))
    assert np.array_equal(_u64(pa), _u64(pb))
    for f in ("final_loss", "validation_mse", "validation_max_error", "final_learning_rate"):
        assert _u64([getattr(ra, f)]) == _u64([getattr(rb, f)]), f
    assert (ra.diverged, ra.halvings, ra.epochs_recorded) == (rb.diverged, rb.halvings, rb.epochs_recorded)
    if lr > 10:
        assert ra.halvings > 0 or ra.diverged  # the runaway / rollback path was exercised
