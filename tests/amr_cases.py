"""End-to-end AMR parity cases shared by the golden generator (reference) and
the GPU tests (product).  Material and initial-condition callables are plain
numpy expressions, evaluated identically by both sides."""
import numpy as np


def _gauss2(x0, y0, beta):
    def ic(X, Y):
        p = np.exp(-beta * ((X - x0) ** 2 + (Y - y0) ** 2))
        z = np.zeros_like(p)
        return np.stack([p, z, z])
    return ic


def _gauss1():
    def ic(x):
        p = np.exp(-100.0 * (x + 1.0) ** 2) + 0.5 * np.exp(-100.0 * (x - 1.5) ** 2)
        return np.stack([p, np.zeros_like(p)])
    return ic


def _swe_ic(X, Y):
    eta = 0.5 * np.exp(-((X - 300.0) ** 2 + (Y - 500.0) ** 2) / 80.0 ** 2)
    z = np.zeros_like(eta)
    return np.stack([eta, z, z])


def _basin(x, y):
    x = np.asarray(x, float)
    y = np.asarray(y, float)
    return -60.0 + 0.09 * x + 10.0 * np.sin(y / 150.0)   # dry beyond x ~ 630


CASES = {
    # C2-like: homogeneous 2D acoustics, adjoint flagging, 3 levels (ratios 2, 2)
    "ac2d_adjoint": dict(
        system="ac", ndim=2, xlim=(-4.0, 4.0), ylim=(-4.0, 4.0), base=(24, 24), ratios=(2, 2),
        material=(lambda x, y: np.full_like(np.asarray(x, float), 4.0),
                  lambda x, y: np.ones_like(np.asarray(x, float))),
        bc=("wall", "wall", "wall", "wall"), ic=_gauss2(0.0, 0.0, 8.0),
        strategy="adjoint", functional=("box", (1.5, 2.5, -2.5, -1.5), (1.0, 0.0, 0.0)),
        window=(2.0, 2.0), adjoint_shape=(32, 32), snapshot_dt=0.1, tol=1e-3,
        regrid_interval=2, buffer=2, efficiency=0.7, max_patch_edge=24, steps=6),
    # heterogeneous 2D acoustics, mixed boundaries, ratios 2 then 4
    "ac2d_hetero": dict(
        system="ac", ndim=2, xlim=(-2.0, 2.0), ylim=(-1.5, 1.5), base=(20, 16), ratios=(2, 4),
        material=(lambda x, y: np.where(np.asarray(y) < 0.3 * np.asarray(x), 4.0, 1.0),
                  lambda x, y: np.where(np.asarray(y) < 0.3 * np.asarray(x), 1.0, 1.5)),
        bc=("outflow", "wall", "wall", "outflow"), ic=_gauss2(-0.5, 0.2, 10.0),
        strategy="adjoint", functional=("box", (1.0, 1.5, -1.0, -0.5), (1.0, 0.0, 0.0)),
        window=(0.8, 1.2), adjoint_shape=(24, 20), snapshot_dt=0.05, tol=1e-3,
        regrid_interval=1, buffer=1, efficiency=0.7, max_patch_edge=32, steps=4),
    # linear shallow water basin with a dry shore, surface flagging
    "swe_basin": dict(
        system="swe", ndim=2, xlim=(0.0, 1000.0), ylim=(0.0, 1000.0), base=(20, 20), ratios=(2,),
        material=_basin, bc=("wall", "wall", "wall", "wall"), ic=_swe_ic,
        strategy="surface", functional=None, window=(0.0, 0.0), tol=0.05,
        regrid_interval=2, buffer=2, efficiency=0.7, max_patch_edge=20, steps=5),
    # C1-like: 1D acoustics across an impedance jump, adjoint flagging, 3 levels
    "ac1d_adjoint": dict(
        system="ac", ndim=1, xlim=(-4.0, 4.0), base=(80,), ratios=(2, 2),
        material=(lambda x: np.where(np.asarray(x) < 0.0, 4.0, 1.0), lambda x: np.ones_like(np.asarray(x, float))),
        bc=("outflow", "outflow"), ic=_gauss1(),
        strategy="adjoint", functional=("box", (1.0, 1.2), (1.0, 0.0)),
        window=(1.5, 1.5), adjoint_shape=(160,), snapshot_dt=0.05, tol=1e-3,
        regrid_interval=1, buffer=3, efficiency=0.7, max_patch_edge=60, steps=6),
    # refine-everywhere equivalence setup (2D)
    "ac2d_everywhere": dict(
        system="ac", ndim=2, xlim=(0.0, 1.0), ylim=(0.0, 1.0), base=(12, 12), ratios=(2,),
        material=(lambda x, y: np.full_like(np.asarray(x, float), 1.0),
                  lambda x, y: np.ones_like(np.asarray(x, float))),
        bc=("wall", "outflow", "outflow", "wall"), ic=_gauss2(0.4, 0.6, 40.0),
        strategy="everywhere", functional=None, window=(0.0, 0.0), tol=0.0,
        regrid_interval=1, buffer=0, efficiency=0.7, max_patch_edge=60, steps=4),
}
