"""The cross-entropy oracle (not in the reference): its analytic
gradients against central finite differences, the reference's own gradient check
(cube3d/reference.hpp:389-405), and the loss against a direct log-softmax."""
import numpy as np

from oracle import cube3d_oracle as O


def test_cross_entropy_oracle_finite_differences():
    rng = np.random.default_rng(3)
    n, h, v = 6, 5, 7
    x = rng.uniform(-1, 1, (n, h))
    w = rng.uniform(-1, 1, (h, v))
    b = rng.uniform(-1, 1, v)
    t = rng.integers(0, v, n)
    loss, cache = O.cross_entropy_fwd(x, w, b, t)
    dx, dw, db = O.cross_entropy_bwd(cache)
    eps = 1e-6
    for arr, grad in ((x, dx), (w, dw), (b, db)):
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = arr[i]
            arr[i] = old + eps
            lp, _ = O.cross_entropy_fwd(x, w, b, t)
            arr[i] = old - eps
            lm, _ = O.cross_entropy_fwd(x, w, b, t)
            arr[i] = old
            assert abs((lp - lm) / (2 * eps) - grad[i]) < 1e-7


def test_cross_entropy_oracle_value_and_shift_invariance():
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (4, 3))
    w = rng.uniform(-1, 1, (3, 5))
    b = rng.uniform(-1, 1, 5)
    t = np.array([0, 4, 2, 2])
    loss, _ = O.cross_entropy_fwd(x, w, b, t)
    logits = x @ w + b
    direct = np.mean(-np.log(np.exp(logits[np.arange(4), t]) / np.exp(logits).sum(1)))
    assert abs(loss - direct) < 1e-12
    # a constant shift of the logits (through the bias) leaves the loss unchanged
    loss2, _ = O.cross_entropy_fwd(x, w, b + 100.0, t)
    assert abs(loss - loss2) < 1e-9
