"""paper_2604_07874_b200 -- B200-native hot path of Valve (arXiv 2604.07874).

The product is libvalve.so (sm_100a CUDA kernels behind the C ABI in include/valve_cuda.h);
`api` mirrors the reference runtime API (colosim) over that ABI.  Importing this package does
not touch the GPU; constructing a pool, gate or selection call does, and fails loudly
(CudaError / ImportError) when the library or the device is missing.

Importing it also asks CUDA for 32 hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS, unless
set): the runtime's streams block on stream memory operations for long stretches (gated launches,
landed-ticket waits), and with the default 8 queues a blocked wait stalls unrelated streams that
share its queue.  It must happen before the process's CUDA context exists (import this package
before the first CUDA call); libvalve.so sets the same default when it is loaded.
"""
import os as _os

_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from .api import (  # noqa: F401
    ChannelController, ChannelLog, CooldownPolicy, CudaError, DevicePool, Gate, HandleState, Hooks,
    InvalidArgument, LogicError, MemoryPool, OutOfRange, ReclaimHandle, ReclaimInstance,
    ReclaimResult, ReservationController, ReservationParams, ValveRuntimeError, copy_params,
    evicted_cost, fifo_reclaim, kernel_launches, oracle_reclaim, selective_reclaim, valve_backend,
)

from .api import LIBVALVE  # noqa: E402,F401
