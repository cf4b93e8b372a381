"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package draws random systems and points and converts high-precision
reals into DD/QD limbs.  It holds none of the method's arithmetic: no
monomial, derivative, Speelpenning or DD/QD arithmetic lives here.
"""
from .systems import (  # noqa: F401
    config_point_rows,
    CONFIGS,
    SystemArrays,
    config_system,
    random_system,
    unit_circle_limbs,
    split_limbs,
    limbs_from_values,
    special_linear_system,
    special_gaussian_system,
    special_univariate_system,
    homogeneous_system,
    system_from_terms,
    homotopy_target,
    real_limbs,
    random_t,
    CommonArrays,
    common_support_system,
    expand_common,
    COMMON_CONFIGS,
    common_config,
    total_degree_homotopy,
    as_common,
)
