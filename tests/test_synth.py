"""Seeded input generators (synth/) — CPU checks: the counter-based config-4 generator reproduces
the published Philox4x32-10 known answers, is shard-invariant, and builds a feasible QP exactly as
BASELINE.json configs[4] prescribes (b = A x0, c = A^T y0 + z0 - q x0, floor(0.3 n) zeros in q)."""
import os

import numpy as np
import torch

from synth import large, make_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_synth_philox_known_answers():
    # Salmon et al. SC'11 / Random123 kat_vectors (tests/golden/philox4x32_10_kat.txt)
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        ctr = [torch.tensor([x], dtype=torch.int64) for x in v[:4]]
        out = large.philox4x32_10(*ctr, v[4], v[5])
        assert [int(o) for o in out] == v[6:10]
        n += 1
    assert n >= 3


def test_normals_stream_offsets_and_moments():
    full = large.normals(4, large.G_ID, 0, 200001)
    for s, c in [(0, 7), (1, 10), (12345, 999), (200000, 1)]:
        assert torch.equal(large.normals(4, large.G_ID, s, c), full[s:s + c])
    z = full.numpy()
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    # different matrix ids / seeds give different streams
    assert not torch.equal(large.normals(4, large.W_ID, 0, 100), large.normals(4, large.H_ID, 0, 100))
    assert not torch.equal(large.normals(4, large.W_ID, 0, 100), large.normals(5, large.W_ID, 0, 100))


def test_config4_shards_reassemble_the_instance():
    m, n = 120, 701
    full = large.generate_shard(m, n, 0, n, chunk_elems=5000)
    parts = [large.generate_shard(m, n, *large.shard_bounds(n, r, 3), chunk_elems=3000) for r in range(3)]
    assert torch.equal(torch.cat([p.At for p in parts]), full.At)
    assert torch.equal(torch.cat([p.c for p in parts]), full.c)
    bsum = sum(p.b_part for p in parts)
    assert torch.allclose(bsum, full.b_part, rtol=1e-13, atol=1e-9)
    # padding rows of the library layout are zero
    assert torch.count_nonzero(full.At[:, m:]) == 0


def test_config4_feasible_point_and_zero_pattern():
    inst = make_config(4, m=200, n=1500, ell=30)
    A = inst.A
    assert np.linalg.norm(A @ inst.x0 - inst.b) <= 1e-13 * np.linalg.norm(inst.b)
    assert np.linalg.norm(A.T @ inst.y0 + inst.z0 - inst.q * inst.x0 - inst.c) <= 1e-13 * np.linalg.norm(inst.c)
    assert int((inst.q == 0).sum()) == int(0.3 * 1500)          # A22
    assert inst.x0.min() >= 0.5 and inst.z0.min() >= 0.5
    # A = W H + 1e-2 G with W, H rank 100: 100 dominant singular values, then the noise level
    s = np.linalg.svd(A, compute_uv=False)
    assert s[99] > 20 * s[100]
    assert 0.5 * 1e-2 * (np.sqrt(1500) - np.sqrt(200)) < s[100] < 2 * 1e-2 * (np.sqrt(1500) + np.sqrt(200))


def test_config4_slice_is_restriction_of_the_generator():
    # A25: the slice QP uses generator columns [0, n) with the same y0 and restricted q, x0, z0
    m, n_gen, n = 100, 900, 300
    full = large.generate_shard(m, n_gen, 0, n_gen, n_gen=n_gen)
    sl = large.generate_shard(m, n, 0, n, n_gen=n_gen)
    assert torch.equal(sl.At, full.At[:n])
    assert torch.equal(sl.q, full.q[:n]) and torch.equal(sl.x0, full.x0[:n]) and torch.equal(sl.y0, full.y0)


def test_make_general_is_strictly_feasible():
    """f1 generator: x0 interior on I and J, z0_F = 0, and (x0, y0, z0, s0) satisfy (P~)/(D~) exactly."""
    from synth import make_general
    inst = make_general(30, 90, 0.2, 0.3, ell=4, seed=3)
    vt, u = inst.extra["vtype"], inst.extra["ub"]
    I, F, J = vt == 0, vt == 1, vt == 2
    assert vt.dtype == np.int8 and F.sum() == 18 and J.sum() == 27
    assert np.all(inst.x0[I] > 0) and np.all(inst.x0[J] > 0) and np.all(inst.x0[J] < u[J])
    assert np.all(inst.z0[F] == 0) and np.all(inst.z0[~F] > 0) and np.all(u[~J] == 0)
    s0 = inst.extra["s0"]
    assert np.allclose(inst.A @ inst.x0, inst.b, atol=1e-12)
    assert np.allclose(inst.c + inst.q * inst.x0 - inst.A.T @ inst.y0 - inst.z0 + s0, 0, atol=1e-12)
    again = make_general(30, 90, 0.2, 0.3, ell=4, seed=3)
    assert np.array_equal(again.A, inst.A) and np.array_equal(again.extra["vtype"], vt)


def test_paper_formulation_generators():
    """App. C.2 dual SVM and App. C.1 portfolio in structure-2 form: shapes, identity blocks, and a
    strictly feasible primal point of the portfolio (x = 1/n, y = F^T x, t = u - M x > 0)."""
    from synth import make_portfolio, make_svm_dual, structured_dense_A
    sv = make_svm_dual(40, 12, tau=2.0)
    A = structured_dense_A(sv.extra["B"], sv.extra["unit_blocks"], sv.m)
    assert A.shape == (13, 52) and np.array_equal(A[:12, 40:], np.eye(12)) and np.all(A[12, 40:] == 0)
    yl = sv.extra["labels"]
    assert np.array_equal(A[12, :40], yl) and np.all(sv.c[:40] == -1) and np.all(sv.q[40:] == 1)
    assert np.all(sv.extra["ub"][:40] == 2.0) and np.all(sv.extra["vtype"][40:] == 1)
    pf = make_portfolio(50, 7, 3)
    A = structured_dense_A(pf.extra["B"], pf.extra["unit_blocks"], pf.m)
    assert A.shape == (11, 60)
    x = np.full(50, 1 / 50)
    FT = -pf.extra["B"][:3]
    y = FT @ x
    t = pf.b[3:10] - pf.extra["B"][3:10] @ x
    assert np.all(t > 0)
    assert np.allclose(A @ np.concatenate([x, y, t]), pf.b, atol=1e-14)


def test_studies_scripts_are_importable():
    """The f4 / Table 3 study scripts import without a GPU (they only touch CUDA inside main())."""
    import importlib
    for name in ("studies.f4_condition", "studies.f4_rank_time", "studies.table3_shapes"):
        mod = importlib.import_module(name)
        assert callable(mod.main)
    from studies.table3_shapes import TABLE3
    assert set(TABLE3) == {"SensIT", "CIFAR10", "RNASeq", "STL-10", "Arcene"}
