"""Seeded synthetic input generators shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the method (no Montgomery multiplication, REDC,
curve arithmetic, gcd or scalar plan).  It only draws numbers: a counter-based splitmix64
stream, Miller-Rabin primality for planting prime factors, and the SURVEY.md §8(d) d1
configuration recipes.  Both sides consume exactly these arrays.
"""
from .gen import (  # noqa: F401
    splitmix64,
    splitmix64_array,
    is_probable_prime,
    random_prime,
    mulmod_inputs,
    sigmas,
    ecm_config,
    ECM_CONFIGS,
    MULMOD_CONFIGS,
    edge_moduli,
    edge_mulmod_inputs,
    near_max_composite,
)
