"""Pins for oracle.sample (NEXT-1 action sampling): SPEC S:L66-67's worked examples and the law of
the draw."""
import numpy as np

from oracle import sample


def test_degenerate_logits_pick_the_max():
    # logits [1000, 0, 0, 0] -> action 0 with log-prob ~ 0
    acts, logp, _ = sample.sample(np.array([[1000.0, 0, 0, 0]] * 64), seed=3, counter=0)
    assert np.all(acts == 0) and np.all(np.abs(logp) < 1e-6)


def test_frequencies_match_softmax():
    # logits [1, 2, 3, 4], 100000 draws -> empirical frequencies within 0.01 of the softmax
    z = np.array([1.0, 2.0, 3.0, 4.0])
    p = np.exp(z - z.max())
    p /= p.sum()
    E = 1000
    counts = np.zeros(4)
    for counter in range(100):
        acts, logp, _ = sample.sample(np.tile(z, (E, 1)), seed=7, counter=counter)
        counts += np.bincount(acts, minlength=4)
        assert np.allclose(logp, np.log(p[acts]), atol=1e-6)
    assert np.all(np.abs(counts / counts.sum() - p) < 0.01)


def test_uniforms_are_uniform_and_keyed():
    u = sample.uniforms(11, 5, 20000)
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.003
    assert not np.array_equal(u[:100], sample.uniforms(11, 6, 100))
    assert not np.array_equal(u[:100], sample.uniforms(12, 5, 100))
    assert np.array_equal(u[:100], sample.uniforms(11, 5, 100))


def test_greedy_is_first_argmax():
    acts, _, _ = sample.sample(np.array([[0.0, 2, 2, 1], [5, 1, 5, 0]]), 0, 0, greedy=True)
    assert list(acts) == [1, 0]
