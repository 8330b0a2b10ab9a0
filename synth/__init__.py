"""Seeded synthetic workloads for the MSPipe node-memory stage.

This package is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2402_15113_b200``).  It draws inputs — event streams,
negatives, edge features, GRU weights — and holds none of the method's
arithmetic (no sampling, dedup, staleness, message, GRU or write-back logic).
"""
from .events import (CONFIGS, WorkloadConfig, edge_features, gru_params, make_events, make_workload,  # noqa: F401
                     node_features, rnn_params, train_params)
