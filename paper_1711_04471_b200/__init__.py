"""paper_1711_04471_b200 — a B200-native 2-D shallow water (2DSW) time step.

The data-parallel hot path of arXiv 1711.04471 §6.2: the
2DSW time loop (predictor ``dyn``, first-order Shapiro filter, velocity
update) fused into one sm_100a CUDA pass behind the C ABI ``include/sw2d.h``
(``libsw2d.so``).  ``sw2d`` is the thin ctypes binding with the C names.
"""
from . import sw2d  # noqa: F401
from .sw2d import (Sw2dError, make_dist, make_params, sw2d_create,  # noqa: F401
                   sw2d_destroy, sw2d_get_state, sw2d_local_rows,
                   sw2d_partition, sw2d_reduce, sw2d_reduce_history,
                   sw2d_set_state, sw2d_step, sw2d_sync)

__all__ = ["sw2d", "Sw2dError", "make_params", "make_dist", "sw2d_create",
           "sw2d_destroy", "sw2d_get_state", "sw2d_local_rows", "sw2d_partition",
           "sw2d_reduce", "sw2d_reduce_history", "sw2d_set_state", "sw2d_step",
           "sw2d_sync"]
