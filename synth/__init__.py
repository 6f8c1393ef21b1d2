"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no operator, no FFT, no
compression, no restoration).  It only states the five BASELINE.json
workload configurations and draws the CN(0,1) box signatures that stand in
for the aggregated far-field patterns A_v(k_p) of PAPER.md eq. (4),
plus synthetic basis functions (box membership, points, CN(0,1) far-field
patterns and currents) for the aggregation / disaggregation steps around the
translation.

Both `oracle/` and `paper_2010_00520_b200/` may import it; neither imports
the other.
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    Basis,
    basis,
    basis_seed,
    currents,
    patterns,
    SEED_BASE,
    Config,
    config,
    signature_seed,
    signatures,
    weights_seed,
)
