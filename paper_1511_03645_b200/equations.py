"""Equation sets and materials (host descriptors of the K1 kernel variants).

Mirrors the reference's plugin surface (equations.py:20-74, 356-534 of
/root/reference/pkg/src/adjamr): materials are sampled on the host from
arbitrary Python callables, then live in HBM as aux planes; the equation
class only selects the kernel template (system, Riemann form, time
reversal).  The interface Riemann and transverse solvers themselves are
inlined in the CUDA step kernels (csrc/k1_exact.cu, csrc/k1_fast.cu).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


class InvalidMaterialError(ValueError):
    """Nonpositive bulk modulus, density, or other bad material data."""


class DryCellError(ValueError):
    """A shallow-water Riemann solve was asked to use a dry cell."""


@dataclass(frozen=True)
class AcousticsMaterial:
    bulk: np.ndarray
    rho: np.ndarray
    c: np.ndarray
    z: np.ndarray

    @classmethod
    def create(cls, bulk, rho) -> "AcousticsMaterial":
        bulk = np.asarray(bulk, dtype=float)
        rho = np.asarray(rho, dtype=float)
        if np.any(bulk <= 0) or np.any(rho <= 0):
            raise InvalidMaterialError("bulk modulus and density must be positive")
        c = np.sqrt(bulk / rho)
        return cls(bulk=bulk, rho=rho, c=c, z=rho * c)

    def __getitem__(self, sl) -> "AcousticsMaterial":
        return AcousticsMaterial(self.bulk[sl], self.rho[sl], self.c[sl], self.z[sl])

    def planes(self) -> list[np.ndarray]:
        """Device aux plane order {c, z, rho, bulk} (include/adjamr_b200.h)."""
        return [self.c, self.z, self.rho, self.bulk]


@dataclass(frozen=True)
class SweMaterial:
    bathymetry: np.ndarray
    depth: np.ndarray
    wet: np.ndarray
    c: np.ndarray
    gravity: float

    @classmethod
    def create(cls, bathymetry, sea_level: float, gravity: float) -> "SweMaterial":
        b = np.asarray(bathymetry, dtype=float)
        depth = sea_level - b
        return cls(bathymetry=b, depth=depth, wet=depth > 0.0,
                   c=np.sqrt(gravity * np.maximum(depth, 0.0)), gravity=gravity)

    def __getitem__(self, sl) -> "SweMaterial":
        return SweMaterial(self.bathymetry[sl], self.depth[sl], self.wet[sl], self.c[sl], self.gravity)

    def planes(self) -> list[np.ndarray]:
        """Device aux plane order {c, depth} (wet <=> depth > 0)."""
        return [self.c, self.depth]


class MaterialModel:
    def sample(self, x, y=None):
        raise NotImplementedError


class AcousticsMaterialModel(MaterialModel):
    def __init__(self, bulk_fn, rho_fn):
        self.bulk_fn = bulk_fn
        self.rho_fn = rho_fn

    def sample(self, x, y=None):
        if y is None:
            return AcousticsMaterial.create(self.bulk_fn(x), self.rho_fn(x))
        return AcousticsMaterial.create(self.bulk_fn(x, y), self.rho_fn(x, y))


class SweMaterialModel(MaterialModel):
    def __init__(self, bathymetry_fn, sea_level: float = 0.0, gravity: float = 9.81):
        self.bathymetry_fn = bathymetry_fn
        self.sea_level = sea_level
        self.gravity = gravity

    def sample(self, x, y=None):
        return SweMaterial.create(self.bathymetry_fn(x, y), self.sea_level, self.gravity)


class EquationSet:
    """One hyperbolic system bound to a material model (equations.py:388-420)."""

    name: str
    m: int
    form: str = "wave"
    is_swe = False
    system: int = -1          # _lib.SYS_*

    def __init__(self, material: MaterialModel):
        self.material = material

    def sample_material(self, x, y=None):
        return self.material.sample(x, y)

    def normal_component(self, axis: int) -> int:
        return 1 if self.m == 2 else 1 + axis

    def max_speed(self, mat):
        return mat.c

    def adjoint(self) -> "EquationSet":
        raise NotImplementedError

    # kernel selection ------------------------------------------------------
    @property
    def reversed_flag(self) -> bool:
        return False

    def kernel_spec(self) -> tuple[int, int, int]:
        """(system, form, reversed) for AdjStepArgs."""
        form = _lib.FORM_FWAVE if self.form == "fwave" else _lib.FORM_WAVE
        return self.system, form, int(self.reversed_flag)

    @property
    def gravity(self) -> float:
        return float(getattr(self.material, "gravity", 0.0))

    @property
    def naux(self) -> int:
        return 2 if self.is_swe else 4


class Acoustics1D(EquationSet):
    name = "acoustics-1d"
    m = 2
    system = _lib.SYS_AC1D

    def adjoint(self):
        return AdjointAcoustics1D(self.material)


class Acoustics2D(EquationSet):
    name = "acoustics-2d"
    m = 3
    system = _lib.SYS_AC2D

    def adjoint(self):
        return AdjointAcoustics2D(self.material)


class SweLinear2D(EquationSet):
    name = "swe-linear-2d"
    m = 3
    is_swe = True
    system = _lib.SYS_SWE2D

    def adjoint(self):
        return AdjointSweLinear2D(self.material)


class _AdjointBase(EquationSet):
    form = "fwave"

    def reversed(self) -> "TimeReversed":
        return TimeReversed(self)


class AdjointAcoustics1D(_AdjointBase):
    name = "adjoint-acoustics-1d"
    m = 2
    system = _lib.SYS_AC1D


class AdjointAcoustics2D(_AdjointBase):
    name = "adjoint-acoustics-2d"
    m = 3
    system = _lib.SYS_AC2D


class AdjointSweLinear2D(_AdjointBase):
    name = "adjoint-swe-linear-2d"
    m = 3
    is_swe = True
    system = _lib.SYS_SWE2D


class TimeReversed(EquationSet):
    """Flux-negated wrapper (equations.py:496-534); selects REV kernels."""

    def __init__(self, inner: EquationSet):
        super().__init__(inner.material)
        self.inner = inner
        self.name = inner.name + "-reversed"
        self.m = inner.m
        self.form = inner.form
        self.is_swe = inner.is_swe
        self.system = inner.system

    @property
    def reversed_flag(self) -> bool:
        return not self.inner.reversed_flag

    def sample_material(self, x, y=None):
        return self.inner.sample_material(x, y)

    def normal_component(self, axis):
        return self.inner.normal_component(axis)

    def max_speed(self, mat):
        return self.inner.max_speed(mat)
