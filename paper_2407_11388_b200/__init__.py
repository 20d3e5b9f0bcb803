"""paper_2407_11388_b200 -- Recurrent Arc Consistency (arXiv 2407.11388) on B200.

The product is librac.so (C ABI, include/rac.h): CUDA kernels for sm_100a that
pack binary relations into per-(x,a) support masks and run the RAC recurrence
(Eq. 1, lines 89-99) to the arc-consistent fixpoint on the device.
``paper_2407_11388_b200.rac`` is the ctypes binding; ``dist`` holds the
multi-process plumbing (NCCL unique-id broadcast over torch.distributed).
"""
from .rac import (RAC_EINVAL, RAC_FULL_FIXPOINT, RAC_OK, RAC_WIPEOUT, RacContext, RacError,  # noqa: F401
                  rac_get_nccl_unique_id, rac_shard_range)
