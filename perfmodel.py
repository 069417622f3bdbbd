"""Byte and flop model of one coarse-Dslash apply.

flops / site  = 9 * (8 N^2 - 2 N) + 8 * 2 N       9 complex mat-vecs + 8 vector adds (R16)
metric bytes  = 9 link matrices + 9 vector records per site, each stored record with its
                fp16 scale (BASELINE.json north_star "bytes = 9 link matrices plus 9 vectors
                per site"; R15)
compulsory    = 9 link matrices + 1 vector read + 1 vector write per site
"""


def flops_per_site(nvec: int) -> int:
    N = 2 * nvec
    return 9 * (8 * N * N - 2 * N) + 8 * 2 * N


def metric_bytes_per_site(nvec: int, prec: str) -> int:
    N = 2 * nvec
    if prec == "fp32":
        return 9 * N * N * 8 + 9 * N * 8
    if prec == "fp16":
        return 9 * (N * N * 4 + 4) + 9 * (N * 4 + 4)
    if prec == "fp64":
        return 9 * N * N * 16 + 9 * N * 16
    raise ValueError(prec)


def compulsory_bytes_per_site(nvec: int, prec: str) -> int:
    N = 2 * nvec
    if prec == "fp32":
        return 9 * N * N * 8 + 2 * N * 8
    if prec == "fp16":
        return 9 * (N * N * 4 + 4) + 2 * (N * 4 + 4)
    raise ValueError(prec)


def arithmetic_intensity(nvec: int, prec: str) -> float:
    return flops_per_site(nvec) / metric_bytes_per_site(nvec, prec)
