"""paper_2304_13541_b200 -- B200-native batched evaluation of D-STACK's scheduling models.

The product is ``libdstack.so`` (C-ABI in include/dstack.h, sm_100a kernels in csrc/); this package
is its thin Python binding.  Importing it fails loudly when the library has not been built.
"""
from . import dstack  # noqa: F401
from .dstack import (DeviceProblem, DstackError, Workspace, alloc_outputs, batch_opt, eval_batch,  # noqa: F401
                     from_device_dict, from_host, knee, schedule_cycle, wmaxmin)

__all__ = ["dstack", "DeviceProblem", "DstackError", "Workspace", "alloc_outputs", "batch_opt", "eval_batch",
           "from_device_dict", "from_host", "knee", "schedule_cycle", "wmaxmin"]
