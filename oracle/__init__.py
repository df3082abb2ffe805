"""CPU oracle for the temporally fused LIF path (arXiv 2408.00280).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product package ``paper_2408_00280_b200`` never imports it, and it imports
nothing from the product package (they share only ``snn_synth``, the seeded input
generator, which holds none of the method's arithmetic).

The arithmetic lives in ``lif_oracle.c`` (plain C, fp64, per-time-step loop);
``oracle.py`` is its ctypes wrapper.  See the header of ``lif_oracle.c`` for the
passages each function follows and DESIGN.md "Readings" for every reading taken
where PAPER.md is silent.
"""
from .oracle import (  # noqa: F401
    OracleParams,
    build_oracle,
    forward,
    backward,
    surrogate,
    smooth_step,
    affine_input,
    affine_grads,
)
