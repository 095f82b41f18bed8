import functools
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_names():
    return sorted(n for n in os.listdir(GOLDEN) if n.endswith(".json"))


def csr(adj, n):
    off = np.zeros(n + 1, np.int64)
    for u, row in enumerate(adj):
        off[u + 1] = off[u] + len(row)
    nb = np.array([v for row in adj for v in row], np.int32)
    return off, nb


def instance_from_golden(g):
    """A full instance dict (the arrays pa_build / the oracle take) for a golden fixture."""
    x = np.array(g["x"], np.float32)
    n, D = x.shape
    off, nb = csr(g["adjacency"], n)
    pool = np.array(g["fes"]["pool"], np.int32)
    return dict(metric=g["metric"], N=n, D=D, dp=D, sub_offsets=off, sub_neighbors=nb,
                member_flags=np.ones(n, np.uint8), reduced=x.copy(), rotated=x.copy(),
                basis=np.array(g["V"], np.float32),
                fes_centroids=np.array(g["fes"]["centroids"], np.float32),
                fes_cell_off=np.array([0, pool.size], np.int64), fes_pool_ids=pool,
                full_offsets=off, full_neighbors=nb,
                queries=np.array([g["query"]], np.float32))


@functools.lru_cache(maxsize=None)
def cached_instance(name, **over):
    import datagen as dg
    cfg = dg.get_config(name, **over)
    return dg.build_instance(cfg)


@pytest.fixture(scope="session")
def c0():
    return cached_instance("C0")


@pytest.fixture(scope="session")
def s1():
    return cached_instance("S1")


@pytest.fixture(scope="session")
def s2():
    return cached_instance("S2")


GOLDEN23 = os.path.join(ROOT, "tests", "golden23")


def golden23_names():
    return sorted(n for n in os.listdir(GOLDEN23) if n.endswith(".json"))


def load_golden23(name):
    with open(os.path.join(GOLDEN23, name)) as f:
        return json.load(f)


def instance_from_golden23(g):
    """Stages ②③ goldens: separate subgraph / full graph, member flags, d' < D."""
    x = np.array(g["x"], np.float32)
    n, D = x.shape
    dp = g["dp"]
    soff, snb = csr(g["sub_adjacency"], n)
    foff, fnb = csr(g["full_adjacency"], n)
    pool = np.array(g["fes"]["pool"], np.int32)
    return dict(metric=g["metric"], N=n, D=D, dp=dp, sub_offsets=soff, sub_neighbors=snb,
                member_flags=np.array(g["members"], np.uint8), reduced=np.ascontiguousarray(x[:, :dp]),
                rotated=x.copy(), basis=np.array(g["V"], np.float32),
                fes_centroids=np.array(g["fes"]["centroids"], np.float32),
                fes_cell_off=np.array([0, pool.size], np.int64), fes_pool_ids=pool,
                full_offsets=foff, full_neighbors=fnb, queries=np.array([g["query"]], np.float32))
