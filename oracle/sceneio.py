"""Oracle (TEST INFRASTRUCTURE ONLY): scene identity / wire format -- SURVEY
§8f row 3.  Only tests/ may import this module.

  rle_encode / rle_decode   jsonio.py:42-60 (run starts where the value changes)
  canonical_dumps           jsonio.py:29-30 (sorted keys, compact separators)
  content_hash              jsonio.py:37-39 (SHA-256 of the canonical UTF-8 bytes)

Pinned against tests/golden/sceneio.json (oracle/make_golden_sceneio.py):
the reference's own scene JSON texts and scene hashes.
"""

import hashlib
import json

import numpy as np


def rle_encode(values):
    """Scalar restatement: one pass, a new run wherever the value changes."""
    out = []
    for v in np.asarray(values).ravel().tolist():
        if out and out[-2] == v:
            out[-1] += 1
        else:
            out += [int(v), 1]
    return out


def rle_decode(pairs, dtype=np.uint8):
    vals = np.asarray(pairs[0::2], dtype=dtype)
    return np.repeat(vals, np.asarray(pairs[1::2], dtype=np.int64))


def canonical_dumps(obj):
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), allow_nan=False)


def content_hash(obj):
    return hashlib.sha256(canonical_dumps(obj).encode("utf-8")).hexdigest()
