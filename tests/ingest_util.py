"""Random on-disk corpora for the ingestion tests (test infrastructure)."""
import os

from oracle import oracle as O


def random_tree(root, seed, nfiles=12, max_len=3000, newline_rate=0.05, depth=2):
    """Writes files (some empty, some in nested directories, some with and
    some without a trailing newline) under root; returns root."""
    rng = O.Mt64(seed)
    os.makedirs(root, exist_ok=True)
    dirs = [root]
    for d in range(depth):
        sub = os.path.join(dirs[-1], f"d{d}")
        os.makedirs(sub, exist_ok=True)
        dirs.append(sub)
    for i in range(nfiles):
        n = rng() % (max_len + 1) if i % 5 else 0
        b = bytearray(rng() % 256 for _ in range(n))
        for j in range(n):
            if rng() % 1000 < newline_rate * 1000:
                b[j] = 10
        if n and i % 3 == 0:
            b[-1] = 10
        d = dirs[rng() % len(dirs)]
        with open(os.path.join(d, f"f{rng() % 1000:03d}_{i}.bin"), "wb") as f:
            f.write(bytes(b))
    return root
