"""The five BASELINE.json configs as seeded synthetic generators.

Generator definitions are shared bit-for-bit by the device generators
(csrc/tl_build.cu) and the CPU checker (oracle/trilist_oracle.c):

* draw(seed, k) = fmix64(seed + (k+1) * 0x9E3779B97F4A7C15), the k-th output of
  the reference's sequential splitmix64 (ordering.cpp:13-19).
* ER: u = (d >> 32) % n, v = (d & 0xFFFFFFFF) % n  (acceptance.cpp:305-316).
* R-MAT: per level one draw against floor(p * 2^64) thresholds for
  (a, b, c, d) = (.57, .19, .19, .05), MSB first, then a seeded bijection on
  `scale` bits scrambles ids.
* Chung-Lu: host-computed fixed-point weight prefix, endpoints by
  upper_bound(prefix, draw % total).

Every config is normalised by Graph::from_edges semantics (self-loops dropped,
duplicates collapsed) and oriented by the (degree, id) order.
"""
from __future__ import annotations

CONFIGS = {
    "c1": dict(name="er_n65536_m1048576", kind="er", n=1 << 16, npairs=1 << 20, seed=1,
               desc="Erdos-Renyi G(n=65,536, m=1,048,576)"),
    "c2": dict(name="rmat_s20_ef16", kind="rmat", scale=20, n=1 << 20, npairs=16 << 20, seed=2,
               desc="R-MAT scale 20, edge factor 16, (.57,.19,.19,.05), ids permuted"),
    "c3": dict(name="chunglu_n2^24_avg32_g2.1", kind="chung_lu", n=1 << 24, avg=32.0, gamma=2.1,
               npairs=(1 << 24) * 16, seed=3,
               desc="Chung-Lu n=2^24, average degree 32, Pareto exponent 2.1, cap sqrt(n*avg)"),
    "c4": dict(name="rmat_s26_ef16", kind="rmat", scale=26, n=1 << 26, npairs=16 << 26, seed=4,
               desc="R-MAT scale 26, edge factor 16"),
    "c5": dict(name="rmat_s28_ef16", kind="rmat", scale=28, n=1 << 28, npairs=16 << 28, seed=5,
               desc="Kronecker/R-MAT scale 28, edge factor 16"),
}


def scaled(cfg_key: str, scale_down: int = 0) -> dict:
    """A smaller instance of the same generator family (for parity tests):
    R-MAT scale - scale_down, ER/Chung-Lu n >> scale_down with the same
    average degree."""
    c = dict(CONFIGS[cfg_key])
    if scale_down <= 0:
        return c
    if c["kind"] == "rmat":
        c["scale"] -= scale_down
        c["n"] = 1 << c["scale"]
        c["npairs"] = 16 << c["scale"]
    else:
        c["n"] >>= scale_down
        c["npairs"] >>= scale_down
    c["name"] = f"{c['name']}_down{scale_down}"
    return c
