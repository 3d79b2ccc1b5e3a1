"""The five workloads of BASELINE.json ``configs`` as plain records.

Parameter names follow the paper's Alfven-like operator (Sec. 1, eq. for L_A):
nu (mass weight), beta (div weight, multiplied by lambda), lambda (Alfven length),
b0 (unit field direction).  ``levels=0`` means "as many levels as the coarsening rule
allows" (reading R6); config 0 asks for an explicit 2-level V-cycle.
"""
from dataclasses import dataclass, field, replace
import math


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    p: int
    n: int
    nu: float
    beta: float
    lam: float
    b0: tuple
    rhs: str            # "uniform" (U[-1,1]) or "normal" (standard normal)
    seed: int = 0
    levels: int = 0     # 0 = automatic coarsening rule
    tol: float = 1e-8

    @property
    def m(self) -> int:
        """Interior B-splines per direction, n+p-2 (Sec. 3.1, space S^p_n)."""
        return self.n + self.p - 2

    @property
    def ndof(self) -> int:
        return self.dim * self.m ** self.dim

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


_S2 = 1.0 / math.sqrt(2.0)
_S3 = 1.0 / math.sqrt(3.0)

CONFIGS = [
    Config("2d_p2_n16", 2, 2, 16, 1.0, 1e-2, 1.0, (1.0, 0.0), "uniform", seed=0, levels=2),
    Config("2d_p3_n256", 2, 3, 256, 1e-2, 1e-3, 1.0, (_S2, _S2), "uniform", seed=1),
    Config("2d_p5_n1024", 2, 5, 1024, 1e-4, 1e-4, 1.0, (1.0, 0.0), "normal", seed=2),
    Config("3d_p3_n64", 3, 3, 64, 1.0, 1e-2, 1.0, (0.0, 0.0, 1.0), "uniform", seed=3),
    Config("3d_p4_n160", 3, 4, 160, 1e-3, 1e-4, 1.0, (_S3, _S3, _S3), "normal", seed=4),
]


def config(i_or_name) -> Config:
    if isinstance(i_or_name, int):
        return CONFIGS[i_or_name]
    for c in CONFIGS:
        if c.name == i_or_name:
            return c
    raise KeyError(i_or_name)
