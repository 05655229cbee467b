"""Host-side seeded draws with the reference's exact streams.

The reference derives every random choice from (seed, *labels) through
numpy's SeedSequence -> PCG64 -> ziggurat normals (seeding.py:11-24).  The
B200 path needs two of those streams, once per plan, never per step:

* the warm-start Q init, `derive_rng(seed, "warm_start_init", param_index)
  .standard_normal((m, r))` (compressors.py:362-367, 43-45), and
* the degenerate-column replacement vectors of Gram-Schmidt,
  `SeedSequence([0x67736673, j, attempt])` (linalg.py:17, 54-58).

Both are drawn here with numpy (the same generator, so bit-identical) and
uploaded to the GPU once; every per-step operation runs in CUDA.
"""

import numpy as np

GS_REPLACEMENT_TAG = 0x67736673


def _label_entropy(label):
    if isinstance(label, (int, np.integer)):
        if label < 0:
            raise ValueError(f"labels must be non-negative, got {label}")
        return int(label)
    if isinstance(label, str):
        return int.from_bytes(label.encode("utf-8"), "little")
    raise TypeError(f"unsupported label type: {type(label).__name__}")


def derive_rng(seed, *labels):
    """seeding.py:21-24 semantics: a Generator that is a pure function of (seed, labels)."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [_label_entropy(x) for x in labels]
    return np.random.default_rng(np.random.SeedSequence(entropy))


def warm_start_q(seed, param_index, m, r):
    """compressors.py:366 — the initial Q of one parameter, float64 (m, r)."""
    return derive_rng(seed, "warm_start_init", param_index).standard_normal((m, r))


_REPL_CACHE = {}


def replacement_column(n, j, attempt=0):
    """linalg.py:54-58 — seeded unit replacement vector, float64 (n,)."""
    key = (n, j, attempt)
    v = _REPL_CACHE.get(key)
    if v is None:
        rng = np.random.default_rng(np.random.SeedSequence([GS_REPLACEMENT_TAG, j, attempt]))
        v = rng.standard_normal(n)
        v = v / np.sqrt(v @ v)
        if n <= 65536:
            _REPL_CACHE[key] = v
    return v
