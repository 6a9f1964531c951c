"""The five workloads of BASELINE.json:configs (shapes and noise only — no arithmetic).

Inputs are synthetic and seeded: A = X·Y0 + noise·E with X (m x k), Y0 (k x n) and E (m x n)
i.i.d. complex Gaussian (parts N(0, 1/2)) from Philox (docs/RNG.md), the construction of
PAPER.md:112 ("constructing B and P to be Gaussian random matrices ... and setting A = BP") plus
the configs' noise term. Headline seed 1.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    k: int
    l: int
    noise: float
    gpus: tuple

    @property
    def sketch_flops(self) -> float:
        """8 l m n real flops of the complex sketch Y = R A (4 real multiply-adds per complex MAC)."""
        return 8.0 * self.l * self.m * self.n

    @property
    def a_bytes(self) -> int:
        return 16 * self.m * self.n

    def scaled(self, f_m: int, f_n: int, k=None, l=None, name=None) -> "Config":
        """Same structure at reduced size (parity tests the oracle finishes in seconds)."""
        k = k or max(2, self.k // max(f_m, f_n))
        l = l or k + (self.l - self.k)
        return Config(name or f"{self.name}/s", self.m // f_m, self.n // f_n, k, l, self.noise,
                      (1,))


CONFIGS = {
    "C1": Config("C1", 1024, 512, 16, 24, 0.0, (1,)),
    "C2": Config("C2", 8192, 8192, 64, 80, 1e-10, (1,)),
    "C3": Config("C3", 65536, 4096, 128, 144, 1e-12, (1, 2, 4, 8)),
    "C4": Config("C4", 32768, 32768, 512, 528, 1e-8, (1, 2, 4, 8)),
    "C5": Config("C5", 131072, 32768, 256, 272, 1e-10, (8, 2, 4, 1)),
}
HEADLINE_SEED = 1
