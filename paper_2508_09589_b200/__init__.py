"""B200-native all-at-once space-time solver (arxiv 2508.09589 hot path).

The product path is libst.so (hand-written CUDA for sm_100a) behind the C ABI in
include/st.h; `paper_2508_09589_b200.st` is a thin ctypes binding (argument marshalling
only). There is no CPU fallback: importing the binding without the built library raises.
"""
from .st import (  # noqa: F401
    Grid, Materials, BCs, Source, Options, Solver, StError, load_library, TorchHostComm,
    nccl_unique_id, nccl_comm_init, nccl_selftest,
    ST_TIME_CONSTANT, ST_SPACE_TIME, ST_SRC_UNIFORM, ST_SRC_SIN, ST_COMM_NONE, ST_COMM_NCCL, ST_COMM_HOST,
)
from .design import design_loop  # noqa: F401,E402
