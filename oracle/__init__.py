"""CPU oracle for the grouped n:m hot path of STen (arXiv 2304.07613).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- nothing on
the product path (``paper_2304_07613_b200``) may import it, and it imports
nothing from there.  See ``oracle/sten_oracle.c`` for the passages followed.
"""
from .oracle import (  # noqa: F401
    build, lib_path, sparsify, densify, spmm, dense_matmul, energy, max_threads,
    brute_select, nmg_patterns, nmg_chunk, nmg_sparsify, nmg_sparsify_exchange, nmg_densify, nmg_spmm,
    nmg_brute_best_energy,
    same_format, sddmm, mask_check, gelu, bias_act,
)
