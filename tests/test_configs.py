"""Input recipes (synth/) and the closed forms they imply.  CPU only."""
import numpy as np
import pytest

from synth import generators as G


def test_deterministic_and_shapes():
    a = G.config("C2")
    b = G.config("C2")
    assert a.shape == (4096, 2) and a.dtype == np.float32
    assert (a.view(np.uint32) == b.view(np.uint32)).all()
    assert np.abs(a).max() <= 12.0
    assert G.config("C1").shape == (256, 256)
    x = G.config("C4", n=1024)
    assert x.shape == (1024, 64) and np.isfinite(x).all()


def test_c1_open_interval_and_symmetry():
    W = G.config("C1")
    off = ~np.eye(256, dtype=bool)
    assert (W[off] > 0).all() and (W[off] < 1).all()
    assert (W == W.T).all() and (np.diag(W) == 0).all()


def test_c5_exact_duplicates():
    """C5: 131072 rows of which exactly 1311 repeat an earlier row (1%): 129761 distinct rows."""
    X = G.config("C5")
    assert X.shape == (131072, 16)
    assert len(np.unique(X, axis=0)) == 129761
    assert X.min() >= 0 and X.max() < 1


def test_c3_closed_form_all_ones():
    """C3: the weight-1 subgraph is connected, so every minimax path can use weight-1 edges
    only and every off-diagonal APPD entry is exactly 1.0 (SURVEY §8(c) pin 5).  This is
    the closed form the GPU C3 parity test checks against."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    W = G.config("C3")
    assert W.min() == 0 and W.max() == 255
    ones = W == 1
    assert ones.sum(1).min() >= 32
    ncomp, _ = connected_components(csr_matrix(ones), directed=False)
    assert ncomp == 1


def test_splitmix_reference_values():
    """splitmix64 seeded with 1234567: first outputs of the public reference algorithm."""
    z = G.splitmix_block(1234567, 0, 3)
    assert [int(v) for v in z] == [6457827717110365317, 3203168211198807973, 9817491932198370423]
