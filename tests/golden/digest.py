"""SHA-256 digests of a roadmap CSR (test infrastructure, no method arithmetic).

Both sides hash the same byte layouts: row_ptr as little-endian int32, the
16-byte edge record's first word dst | coll << 31 as uint32, and the raw
float32 bits of w, s, c.  make_golden.py hashes the oracle's CSR; the GPU
tests hash mpap_roadmap_export's arrays and compare."""
import hashlib

import numpy as np


def csr_digests(rm) -> dict:
    rp = np.ascontiguousarray(rm["row_ptr"], dtype="<i4")
    dc = (np.asarray(rm["dst"]).astype(np.uint32) | (np.asarray(rm["coll"]).astype(np.uint32) << np.uint32(31)))
    out = {"row_ptr": hashlib.sha256(rp.tobytes()).hexdigest(),
           "dst_coll": hashlib.sha256(np.ascontiguousarray(dc, dtype="<u4").tobytes()).hexdigest()}
    for k in ("w", "s", "c"):
        out[k] = hashlib.sha256(np.ascontiguousarray(rm[k], dtype="<f4").view("<u4").tobytes()).hexdigest()
    return out
