"""B200-native trajectory-manager data plane (SeamlessFlow, arXiv 2508.11553).

Drop-in replacements for the reference's ``rolloutlab.trie.SessionTrie`` and
``rolloutlab.trajectory.TrajectoryManager`` whose session histories live in a
GPU-resident arena and whose longest-prefix matching, recording and trajectory
assembly run as hand-written sm_100a CUDA kernels behind a C ABI
(include/tmstore.h, libtmstore.so).  No CPU fallback: without the built extension
and a GPU the store raises.
"""

from .core import (
    GenParams,
    InvalidParamsError,
    ModelVersion,
    SpanOrigin,
    TokenId,
    TokenSpan,
    Trajectory,
    ValidationReport,
    is_off_policy,
    read_trajectories,
    trajectory_from_record,
    trajectory_to_line,
    trajectory_to_record,
    validate_trajectory,
    version_lag,
    write_trajectories,
)
from .store import DeviceStore, Packed, RecordResult, default_store
from .trajectory import (
    PendingRequest,
    ProxyRetryableError,
    PumpStatus,
    RequestState,
    TrajectoryManager,
    UnknownSessionError,
)
from .trie import InsertResult, SessionTrie, StorageStats, TrieNode

__all__ = [
    "DeviceStore", "GenParams", "InsertResult", "InvalidParamsError", "ModelVersion", "Packed", "PendingRequest",
    "ProxyRetryableError", "PumpStatus", "RecordResult", "RequestState", "SessionTrie", "SpanOrigin", "StorageStats",
    "TokenId", "TokenSpan", "Trajectory", "TrajectoryManager", "TrieNode", "UnknownSessionError", "ValidationReport",
    "default_store", "is_off_policy", "read_trajectories", "trajectory_from_record", "trajectory_to_line",
    "trajectory_to_record", "validate_trajectory", "version_lag", "write_trajectories",
]
__version__ = "0.1.0"
