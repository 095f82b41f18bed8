"""Input generators: structural invariants of what datagen hands to build(),
and its exhaustive-scan ground truth pinned to the oracle's brute force (O11)."""
import numpy as np

import datagen as dg
import oracle as orc


def _csr_ok(off, nb, N, R):
    assert off[0] == 0 and off[-1] == nb.size and np.all(np.diff(off) >= 0)
    assert np.all((nb >= 0) & (nb < N))
    deg = np.diff(off)
    assert deg.max() <= R
    for u in range(0, N, max(1, N // 500)):
        row = nb[off[u]:off[u + 1]]
        assert u not in row and len(set(row)) == len(row)


def test_c0_structure(c0):
    cfg = c0["cfg"]
    N = cfg.N
    _csr_ok(c0["sub_offsets"], c0["sub_neighbors"], N, cfg.R)
    _csr_ok(c0["full_offsets"], c0["full_neighbors"], N, cfg.R)
    flags = c0["member_flags"]
    assert abs(flags.sum() - cfg.ratio * N) <= 0.02 * N
    deg = np.diff(c0["sub_offsets"])
    assert np.all(deg[flags == 0] == 0)                                       # non-members: zero out-degree
    assert np.all(flags[c0["sub_neighbors"]] == 1)                            # no edges into non-members
    V = c0["V64"]
    assert np.abs(V.T @ V - np.eye(cfg.D)).max() < 1e-10
    assert np.all(flags[c0["fes_pool_ids"]] == 1)
    assert np.all(np.diff(c0["fes_cell_off"]) > 0) and c0["fes_cell_off"].size == cfg.r + 1
    assert np.array_equal(c0["reduced"], c0["rotated"][:, :cfg.dp])


def test_sampling_ratio_one_is_all_members():
    off = np.array([0, 1, 2, 3], np.int64)
    nb = np.array([1, 2, 0], np.int32)
    assert dg.sample_members(off, nb, 1.0, 1).sum() == 3


def test_ground_truth_matches_oracle_brute_force(c0):
    """datagen's GT (fp32 scan + fp64 re-rank) == the oracle's exhaustive fp64 brute force."""
    import torch
    cfg = c0["cfg"]
    Qh = orc.project(c0["queries"], c0["basis"])
    bi, bd = orc.brute_force(Qh, c0["rotated"], 10)
    gi, gd = dg.ground_truth(torch.from_numpy(Qh), torch.from_numpy(c0["rotated"]), 10)
    assert np.array_equal(gi, bi)
    np.testing.assert_allclose(gd, bd, rtol=1e-12)
    mem = np.flatnonzero(c0["member_flags"]).astype(np.int32)
    bi, _ = orc.brute_force(Qh, c0["reduced"], 10, ids=mem)
    gi, _ = dg.ground_truth(torch.from_numpy(Qh[:, :cfg.dp]), torch.from_numpy(c0["reduced"]), 10,
                            ids=torch.from_numpy(mem.astype(np.int64)))
    assert np.array_equal(gi, bi)


def test_shaped_ip_structure(s2):
    cfg = s2["cfg"]
    _csr_ok(s2["sub_offsets"], s2["sub_neighbors"], cfg.N, cfg.R)
    assert s2["metric"] == "ip"
    norms = np.linalg.norm(s2["rotated"], axis=1)
    np.testing.assert_allclose(norms, 1.0, rtol=1e-4)                          # normalised base rows


def test_streamed_reduced_rows_match_full_generation():
    """C3/C4's streamed generator (datagen/large.py gen_reduced: the full rows are
    never stored) yields the same reduced rows X_r = (X·V)[:, :d'] as generating X
    whole, fitting V (fit_svd) and rotating it; and the reduced-only instance has
    the GPU stage's structure (members-only subgraph, FES over members, GT_sub)."""
    import torch
    from datagen import large
    cfg = dg.get_config("C3", N=20_000, D=96, dp=32, m=32, n_e=4096)
    Xr, V, Q = large.gen_reduced(cfg, "cpu")
    X, _ = dg.gen_base(cfg, "cpu")
    V0 = dg.fit_svd(X, cfg.seeds["base"])
    np.testing.assert_allclose(np.abs(V[:, :cfg.dp]), np.abs(V0[:, :cfg.dp]), atol=1e-9)
    ref = dg.rotate(X, V0)[:, :cfg.dp]
    np.testing.assert_allclose(Xr.numpy(), ref.numpy(), rtol=1e-5, atol=1e-6)
    assert torch.equal(Q, dg.gen_queries(cfg, "cpu"))
    inst = large.build_instance_reduced(cfg, device="cpu", gt_k=10)
    flags = inst["member_flags"]
    assert abs(flags.sum() - cfg.ratio * cfg.N) <= 0.02 * cfg.N
    _csr_ok(inst["sub_offsets"], inst["sub_neighbors"], cfg.N, cfg.R)
    assert np.all(np.diff(inst["sub_offsets"])[flags == 0] == 0)
    assert np.all(flags[inst["sub_neighbors"]] == 1) and np.all(flags[inst["fes_pool_ids"]] == 1)
    assert "rotated" not in inst and inst["reduced"].shape == (cfg.N, cfg.dp)
    Qh = orc.project(inst["queries"], inst["basis"])
    mem = np.flatnonzero(flags)
    ids, _ = orc.brute_force(Qh[:, :cfg.dp], inst["reduced"], 10, ids=mem)
    assert np.array_equal(ids, inst["gt_sub_ids"][:, :10])


def test_large_instance_cache_is_per_query_count(tmp_path):
    """The graph cache of the 100M tools is shared across query counts, the
    ground truths are not: a second build with a different m (the scaling run's
    N·10K queries after the 1-GPU run's 10K) reuses the graphs and gets the
    ground truth of ITS queries — equal to an uncached build's."""
    from datagen import large
    cfg = dg.get_config("C3", N=12_000, D=64, dp=16, m=8, n_e=2048)
    a = large.build_instance_reduced(cfg, device="cpu", cache=str(tmp_path), gt_k=10)
    cfg2 = dg.get_config("C3", N=12_000, D=64, dp=16, m=12, n_e=2048)
    b = large.build_instance_reduced(cfg2, device="cpu", cache=str(tmp_path), gt_k=10)
    c = large.build_instance_reduced(cfg2, device="cpu", cache=None, gt_k=10)
    assert a["gt_sub_ids"].shape[0] == 8 and b["gt_sub_ids"].shape[0] == 12
    assert np.array_equal(b["gt_sub_ids"], c["gt_sub_ids"])
    assert np.array_equal(b["sub_neighbors"], c["sub_neighbors"])
    b2 = large.build_instance_reduced(cfg2, device="cpu", cache=str(tmp_path), gt_k=10)   # both cached now
    assert np.array_equal(b2["gt_sub_ids"], c["gt_sub_ids"])


def test_large_full_instance_cache_is_per_query_count(tmp_path):
    """Same for the full-vector 100M tool (C2): graphs cached once, GT and GT_sub per m."""
    from datagen import large
    cfg = dg.get_config("C2", N=12_000, D=32, dp=16, m=8, n_e=2048)
    large.build_instance_large(cfg, device="cpu", cache=str(tmp_path), gt_k=10)
    cfg2 = dg.get_config("C2", N=12_000, D=32, dp=16, m=12, n_e=2048)
    b = large.build_instance_large(cfg2, device="cpu", cache=str(tmp_path), gt_k=10)
    c = large.build_instance_large(cfg2, device="cpu", cache=None, gt_k=10)
    for key in ("gt_ids", "gt_sub_ids", "full_neighbors", "sub_neighbors"):
        assert np.array_equal(b[key], c[key]), key
    assert b["gt_ids"].shape[0] == 12
