"""Oracle for SURVEY.md §8 row F2: the feature-fetch stage (PAPER.md P:L189,
stage 2 "Fetch feature"; subgraph shape P:L1153; |d_v|, |d_e| Table
`tab:datasets` P:L391-L395).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this module.  Shares no code with
paper_2402_15113_b200/csrc/features.cu.

The stage is a plain gather, so the oracle is its definition: for every
subgraph slot (r, s), the node-feature row of the subgraph node sub_ids[r, s]
and, for every sampled link, the edge-feature row of its event id; pads (-1)
give zero rows.
"""
from __future__ import annotations

import numpy as np


def feature_fetch(sub_ids, sampled_eids, node_feat=None, edge_feat=None):
    out_n = out_e = None
    if node_feat is not None:
        sub = np.asarray(sub_ids)
        out_n = np.zeros(sub.shape + (node_feat.shape[1],), np.float32)
        ok = sub >= 0
        out_n[ok] = node_feat[sub[ok]]
    if edge_feat is not None:
        eid = np.asarray(sampled_eids)
        out_e = np.zeros(eid.shape + (edge_feat.shape[1],), np.float32)
        ok = eid >= 0
        out_e[ok] = edge_feat[eid[ok]]
    return out_n, out_e
