"""Shared helpers for the test-suite: paths, and a parallel, cached runner for
the fp64 oracle (full-size parity needs dozens of multi-second oracle calls).

The runner only ever calls ``oracle/fllf_oracle.py``; a cached value is an
oracle output written by this module, keyed by the SHA-256 of the oracle's
source, the function name, its keyword arguments and the input arrays, so any
change of the oracle or of an input misses the cache.  Cache directory:
``$FLLF_ORACLE_CACHE`` (default ``~/.cache/fllf_oracle``); ``FLLF_ORACLE_CACHE=off``
disables it.  The cache is an accelerator only: a cold cache recomputes.
"""
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_ORACLE_SRC = os.path.join(ROOT, "oracle", "fllf_oracle.py")


def _cache_dir():
    d = os.environ.get("FLLF_ORACLE_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "fllf_oracle"))
    return None if d == "off" else d


def _key(name, kwargs):
    h = hashlib.sha256()
    h.update(open(_ORACLE_SRC, "rb").read())
    h.update(name.encode())
    for k in sorted(kwargs):
        v = kwargs[k]
        h.update(k.encode())
        if isinstance(v, np.ndarray):
            h.update(str((v.dtype, v.shape)).encode())
            h.update(np.ascontiguousarray(v).tobytes())
        else:
            h.update(repr(v).encode())
    return h.hexdigest()


def _oracle_call(job):
    """Worker: (function name, kwargs) -> oracle output (float64 array)."""
    name, kwargs = job
    from oracle import fllf_oracle as O
    return np.asarray(getattr(O, name)(**kwargs), dtype=np.float64)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def oracle_many(name, jobs):
    """[oracle.<name>(**kw) for kw in jobs], computed in parallel worker
    processes (spawned, single-threaded numpy) and cached on disk."""
    d = _cache_dir()
    keys = [_key(name, kw) for kw in jobs]
    out = [None] * len(jobs)
    todo = []
    for i, k in enumerate(keys):
        p = os.path.join(d, k + ".npy") if d else None
        if p and os.path.exists(p):
            try:
                out[i] = np.load(p)
                continue
            except Exception:
                pass
        todo.append(i)
    if todo:
        if len(todo) == 1:
            res = [_oracle_call((name, jobs[todo[0]]))]
        else:
            import multiprocessing as mp
            for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
                os.environ.setdefault(v, "1")
            with mp.get_context("spawn").Pool(min(host_cores(), len(todo))) as pool:
                res = pool.map(_oracle_call, [(name, jobs[i]) for i in todo], chunksize=1)
        for i, r in zip(todo, res):
            out[i] = r
            if d:
                try:
                    os.makedirs(d, exist_ok=True)
                    tmp = os.path.join(d, f"{keys[i]}.{os.getpid()}.tmp.npy")
                    np.save(tmp, r)
                    os.replace(tmp, os.path.join(d, keys[i] + ".npy"))
                except OSError:
                    pass
    return out
