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
