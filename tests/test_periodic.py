"""Periodic boundaries (an extension for BASELINE C3's periodic x; the
reference has wall and outflow only, so parity is against the oracle's own
restatement: ghosts wrap to the opposite interior, x slabs then y slabs).
CPU: the oracle's wrap and the BoundarySpec rules.  GPU: fill + step of a
periodic-x patch, EXACT bitwise and FAST within 1e-12, and the refusal of
patches that do not span the periodic axis."""
import numpy as np
import pytest

from oracle import adjamr_oracle as O

G = 2


def test_oracle_periodic_wrap():
    rng = np.random.default_rng(0)
    q = rng.standard_normal((3, 12 + 2 * G, 9 + 2 * G))
    out = O.fill_physical(q, G, {"xlo": True, "xhi": True, "ylo": True, "yhi": True},
                          {"xlo": "periodic", "xhi": "periodic", "ylo": "wall", "yhi": "outflow"}, (1, 2))
    inner = out[:, :, G:-G]
    assert np.array_equal(inner[:, :G], inner[:, 12:12 + G])          # low ghosts = last interior rows
    assert np.array_equal(inner[:, -G:], inner[:, G:2 * G])           # high ghosts = first interior rows
    # a periodic step equals the step of the same data with the wrapped rows as an interior halo
    aux = np.stack([np.full(q.shape[1:], 2.0), np.full(q.shape[1:], 2.0), np.ones(q.shape[1:]),
                    np.full(q.shape[1:], 4.0)])
    a, _ = O.step_2d(out, aux, 0.01, 0.1, 0.1, O.AC2D)
    big = np.concatenate([out[:, G:-G][:, -4:], out[:, G:-G], out[:, G:-G][:, :4]], axis=1)
    bigaux = np.stack([np.full(big.shape[1:], v) for v in (2.0, 2.0, 1.0, 4.0)])
    b, _ = O.step_2d(big, bigaux, 0.01, 0.1, 0.1, O.AC2D)
    assert np.array_equal(a[:, G:-G, G:-G], b[:, 4:-4, G:-G])


def test_boundary_spec_periodic_rules():
    from paper_1511_03645_b200 import solver
    solver.BoundarySpec("periodic", "periodic", "wall", "wall")
    with pytest.raises(ValueError):
        solver.BoundarySpec("periodic", "outflow", "wall", "wall")
    with pytest.raises(ValueError):
        solver.BoundarySpec("wall", "wall", "periodic", "wall")


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_periodic_fill_and_step_vs_oracle(variant):
    from paper_1511_03645_b200 import _lib, solver
    from tests.helpers import norm_rel, patch_from_arrays
    rng = np.random.default_rng(1)
    nx, ny = 40, 33
    q = rng.standard_normal((3, nx + 2 * G, ny + 2 * G))
    rho = rng.uniform(0.8, 1.5, q.shape[1:])
    bulk = rng.uniform(1.0, 4.0, q.shape[1:])
    c = np.sqrt(bulk / rho)
    aux = np.stack([c, rho * c, rho, bulk])
    h, p = patch_from_arrays(q, aux, False, 0.1, 0.1)
    from tests.helpers import make_equation
    eq = make_equation("ac2d")
    bc = solver.BoundarySpec("periodic", "periodic", "wall", "outflow")
    var = _lib.VARIANT_EXACT if variant == "exact" else _lib.VARIANT_FAST
    want = np.array(q)
    dt = 0.02
    for _ in range(3):
        solver.fill_ghost_physical(p, bc, eq, (nx, ny))
        solver.step_patch(p, dt, eq, "MC", variant=var)
        want = O.fill_physical(want, G, {"xlo": True, "xhi": True, "ylo": True, "yhi": True},
                               {"xlo": "periodic", "xhi": "periodic", "ylo": "wall", "yhi": "outflow"}, (1, 2))
        want, _ = O.step_2d(want, aux, dt, 0.1, 0.1, O.AC2D)
    got = np.array(p.state)[:, G:-G, G:-G]
    if variant == "exact":
        assert np.array_equal(got, want[:, G:-G, G:-G])
    else:
        assert norm_rel(got, want[:, G:-G, G:-G]) <= 1e-12


@pytest.mark.gpu
def test_periodic_refuses_partial_patches():
    from paper_1511_03645_b200 import solver
    from paper_1511_03645_b200.geometry import Patch, PatchHierarchy
    from tests.helpers import make_equation
    h = PatchHierarchy(xlim=(0.0, 1.0), ylim=(0.0, 1.0), base_shape=(64, 64), ratios=[])
    p = Patch(h.make_spec(1, (0, 0), (31, 63)), 3)
    eq = make_equation("ac2d")
    bc = solver.BoundarySpec("periodic", "periodic", "wall", "wall")
    solver.sample_patch_material(p, eq, bc, (64, 64))
    with pytest.raises(ValueError):
        solver.fill_ghost_physical(p, bc, eq, (64, 64))
