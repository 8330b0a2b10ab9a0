"""MSPipe (arXiv 2402.15113) node-memory stage on B200 (sm_100a).

The product is libmspipe.so (C ABI: include/mspipe.h); this package is its
thin ctypes binding (_C), host-side input preparation (graph) and the
stream-ordered stage driver (stage).  No CPU fallback: every step of the
stage runs in the library's CUDA kernels.
"""
from . import _C  # noqa: F401
from .build import build  # noqa: F401
from .graph import build_tcsr, build_tcsr_host, gamma_quantile  # noqa: F401
from .stage import MemoryStage, StageConfig, schedule_ops, snapshot_versions  # noqa: F401
from .shard import LoopbackShards, ShardRank, key_base, local_range  # noqa: F401
