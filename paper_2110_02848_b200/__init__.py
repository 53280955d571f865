"""B200-native eager WFST composition (arXiv 2110.02848) -- Python binding of libfstc.so.

The compute path is the CUDA library (``csrc/`` -> ``libfstc.so``, C ABI in ``include/fstc.h``);
this package only marshals arguments.  It never imports ``oracle/``.
"""
from .fstc import (FST_COMPOSE_EPS_FILTER, FST_COMPOSE_PROVENANCE, FST_EPS, Comm, Fst, FstError, compose,
                   fst_compose, fst_compose_batch, fst_compose_chain, fst_compose_ex, fst_compose_sharded, fst_compose_sharded_local, fst_create,
                   fst_forward_score, fst_grad_scatter, fst_launch_count, fst_set_profiling, fst_set_tile_mode, fst_set_wave_mode, fst_version, load_library)

__all__ = ["FST_COMPOSE_EPS_FILTER", "FST_COMPOSE_PROVENANCE", "FST_EPS", "Comm", "Fst", "FstError", "compose",
           "fst_compose", "fst_compose_batch", "fst_compose_chain", "fst_compose_ex", "fst_compose_sharded", "fst_compose_sharded_local", "fst_create",
           "fst_forward_score", "fst_grad_scatter", "fst_launch_count", "fst_set_profiling", "fst_set_tile_mode", "fst_set_wave_mode", "fst_version", "load_library"]
