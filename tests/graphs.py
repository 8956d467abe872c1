"""Hand-built and random CSR graphs shared by the oracle pins and the GPU
parity tests (test data only)."""
import numpy as np


def csr(n, edges):
    """edges: list of (u, v, w, s, c[, coll]) -> CSR dict sorted by (u, v)."""
    edges = sorted(edges, key=lambda e: (e[0], e[1]))
    row_ptr = np.zeros(n + 1, np.int32)
    for e in edges:
        row_ptr[e[0] + 1] += 1
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    return dict(n=n, row_ptr=row_ptr,
                dst=np.array([e[1] for e in edges], np.int32),
                w=np.array([e[2] for e in edges], np.float32),
                s=np.array([e[3] for e in edges], np.float32),
                c=np.array([e[4] for e in edges], np.float32),
                coll=np.array([e[5] if len(e) > 5 else 0 for e in edges], np.uint8))


def random_graph(rng, n, deg, neg_frac=0.3):
    edges = []
    for u in range(n):
        vs = rng.choice([v for v in range(n) if v != u], size=min(deg, n - 1), replace=False)
        for v in vs:
            w = float(rng.uniform(0.1, 1.0))
            s = float(rng.uniform(-0.3, 0.5)) if rng.uniform() < neg_frac else float(rng.uniform(0.0, 0.5))
            c = max(0.0, s) if s > 0 else float(rng.uniform(0.0, 0.2))
            edges.append((u, int(v), w, s, c, int(rng.uniform() < 0.1)))
    return csr(n, edges)
