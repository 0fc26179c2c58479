"""Host batch assembly for the feature front end: raw categorical keys, text strings
and item histories -> one table-major CSR of 64-bit keys for cvr_embed_keys.  Text n-grams and history
truncation run in libcvr (cvr_text_ngram_keys / cvr_truncate_bags); this module only concatenates the
per-table CSRs (argument marshalling).  Hashing and pooling happen on the GPU inside the gather kernel."""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from ._cvr import text_ngram_keys, truncate_bags


def feature_spec(cfg, spec) -> Tuple[List[int], List[int]]:
    """(vocab, pool_mode) for cvr_set_feature_spec: every table hashed with vocab = rows - 1 (the last row is
    the `unseen' row); categorical tables sum, text and history tables mean-pool."""
    vocab = [int(r) - 1 for r in cfg.rows]
    mode = [0 if k == "cat" else 1 for k in spec["kinds"]]
    return vocab, mode


def assemble_keys(fb, spec) -> Tuple[np.ndarray, np.ndarray]:
    """FeatureBatch -> (keys int64 [nnz] (uint64 bit patterns), offsets int32 [T*B + 1]), table-major."""
    parts, lens = [], []
    for kind, tab in zip(spec["kinds"], fb.tables):
        if tab[0] == "text":
            k, o = text_ngram_keys(tab[1], spec["ngram"])
        else:
            k, o = tab[1], tab[2]
            if kind == "seq":
                k, o = truncate_bags(k, o, spec["max_len"])
        parts.append(np.asarray(k, np.uint64))
        lens.append(np.diff(o.astype(np.int64)))
    keys = np.concatenate(parts) if parts else np.zeros(0, np.uint64)
    off = np.zeros(sum(len(x) for x in lens) + 1, np.int64)
    off[1:] = np.cumsum(np.concatenate(lens))
    return keys.view(np.int64), off.astype(np.int32)
