"""End-to-end parity of the encrypted bi-branch forward on the GPU engine
against the reference's own outputs (tests/golden/*.npz, generated from
/root/reference by tests/golden/make_golden.py):

  * OpRecorder counts and per-layer tables: identical integers;
  * decrypted logits vs the reference's float64 `reference_forward`:
    |diff| <= LOGIT_TOL (CKKS is approximate; the measured error is printed)
    and 100% argmax agreement.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

import paper_2402_01296_b200 as B  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402
from paper_2402_01296_b200.network import DecomposedInput  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOGIT_TOL = 1e-6   # absolute, Delta = 2^50, 50-bit rescale primes


def _load(name):
    d = np.load(os.path.join(GOLD, name + ".npz"))
    w = TensorArchive({k[3:]: d[k] for k in d.files if k.startswith("w::")})
    dec = [DecomposedInput(s, f, (0, 0, s.shape[-2], s.shape[-1])) for s, f in zip(d["sens"], d["full"])]
    return d, w, dec, json.loads(str(d["meta"]))


def _check(logits, ref, tol=LOGIT_TOL):
    err = np.abs(logits - ref).max()
    print(f"max |logit - reference| = {err:.3e}")
    assert err <= tol
    assert (logits.argmax(1) == ref.argmax(1)).all()


def test_cnn3_fixture_bhw_matches_reference():
    d, w, dec, meta = _load("cnn3_fixture")
    bundle = B.get("cnn3")
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="bhw")
    assert res.recorder.snapshot() == meta["counts_bhw"]
    assert [list(x) for x in res.recorder.layer_table()] == meta["layer_table"]
    assert res.logits_ct.level == 1
    _check(res.decrypt_logits(), d["logits_ref"])
    assert B.taint_check(bundle.bi, res.recorder).passed


def test_cnn3_backbone_fully_encrypted_matches_reference():
    """forward_backbone (the fully-encrypted single-chain baseline, SURVEY 8(f)
    item 3): the reference's counts (1952 HE ops) and per-layer table as
    integers, logits vs reference_backbone, and taint_check failing on every
    op-bearing layer as in the reference (pkg/tests/test_network.py:247-256, 325-333)."""
    d = np.load(os.path.join(GOLD, "cnn3_backbone.npz"))
    meta = json.loads(str(d["meta"]))
    w = TensorArchive({k[3:]: d[k] for k in d.files if k.startswith("w::")})
    bundle = B.get("cnn3")
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_backbone(bundle.backbone, d["image"][None], w, ctx, strategy="hw")
    c = res.recorder.snapshot()
    assert c == meta["counts_hw"]
    assert c["Add_PC"] + c["Add_CC"] + c["Mul_PC"] + c["Mul_CC"] == 1952
    assert [list(x) for x in res.recorder.layer_table()] == meta["layer_table"]
    _check(res.decrypt_logits(), d["logits_ref"])
    assert not B.taint_check(bundle.backbone, res.recorder).passed


def test_cnn3_hw_single_image_counts():
    d, w, dec, meta = _load("cnn3_fixture")
    bundle = B.get("cnn3")
    ctx = B.make_context(1 << 13, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, dec[0], w, ctx, strategy="hw")
    assert res.recorder.snapshot() == meta["counts_hw"]
    _check(res.decrypt_logits(), d["logits_ref"][:1])


def test_cnn3_config1_matches_reference():
    d, w, dec, meta = _load("cnn3_cfg1")
    bundle = B.get("cnn3")
    ctx = B.make_context(8192, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="hw")
    assert res.recorder.snapshot() == meta["counts_hw"]
    _check(res.decrypt_logits(), d["logits_ref"])


def test_cifar3_config4_matches_reference():
    d, w, dec, meta = _load("cifar3_cfg4")
    bundle = B.get("cifar3")
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="bhw")
    assert res.recorder.snapshot() == meta["counts_bhw"]
    assert [list(x) for x in res.recorder.layer_table()] == meta["layer_table"]
    _check(res.decrypt_logits(), d["logits_ref"])


def test_cifar3_group_batching_equals_single_sets():
    d, w, dec, meta = _load("cifar3_cfg4")
    bundle = B.get("cifar3")
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, dec[:7], w, ctx, strategy="bhw", group_size=3)   # G = 3, last padded
    assert res.logits_ct.batch == 3
    assert res.recorder.snapshot() == meta["counts_bhw"]   # one op set, independent of G
    logits = res.decrypt_logits()
    assert logits.shape == (7, 10)
    _check(logits, d["logits_ref"][:7])


def test_graphed_single_image_forward_matches_reference():
    """CUDA-graph replay of the cnn3 1-image forward (config 1): fresh
    encryption randomness per replay, same logits as the reference."""
    from paper_2402_01296_b200.graphs import GraphedForward

    d, w, dec, meta = _load("cnn3_cfg1")
    bundle = B.get("cnn3")
    ctx = B.make_context(8192, B.required_levels(bundle) + 1, 2.0 ** 50)
    gf = GraphedForward(bundle.bi, w, ctx, (1, 1, 14, 14), (1, 1, 28, 28), strategy="hw")
    assert gf.recorder.snapshot() == meta["counts_hw"]
    out1 = gf(d["sens"], d["full"])
    _check(out1, d["logits_ref"])
    d2, w2, dec2, _ = _load("cnn3_fixture")          # different inputs, same graph
    sens2 = d2["sens"][:1]
    full2 = d2["full"][:1]
    ref2 = B.reference_forward(bundle.bi, [DecomposedInput(sens2[0], full2[0], (7, 7, 14, 14))], w)
    _check(gf(sens2, full2), ref2)
    out3 = gf(d["sens"], d["full"])
    _check(out3, d["logits_ref"])
    assert not np.array_equal(out1, out3)            # fresh encryption noise on every replay


@pytest.mark.parametrize("n1,n2,tiles", [(4, 2, 1), (30, 7, 1), (125, 50, 1), (40, 10, 4)])
def test_fc_bsgs_matches_direct_and_plain(n1, n2, tiles, monkeypatch):
    """fc_forward (layers.py:275-324) by baby-step/giant-step vs the direct
    per-diagonal lazy sum: same reference counts, same values (to CKKS noise)."""
    rng = np.random.default_rng(n1 * 31 + n2)
    ctx = B.make_context(2048, 3, 2.0 ** 50)
    S = ctx.slot_count
    step = 256 if tiles > 1 else 0
    xs = rng.standard_normal((tiles, n1))
    slots = np.zeros(S)
    for tt in range(tiles):
        slots[tt * step:tt * step + n1] = xs[tt]
    W = rng.standard_normal((n1, n2)) / np.sqrt(n1)
    kb = rng.standard_normal(n2)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BCN_FC_BSGS", mode)
        rec = B.OpRecorder()
        ct = B.encrypt_vector(slots, ctx)
        out = B.fc_forward(ct, W, kb, ctx, rec, tiles=tiles, tile_step=step)
        dec = B.decrypt_vector(out, ctx)
        res[mode] = (np.stack([dec[tt * step:tt * step + n2] for tt in range(tiles)]), rec.snapshot(), out.level)
    want = xs @ W + kb
    for mode, (got, counts, level) in res.items():
        assert np.abs(got - want).max() < 1e-8, mode
        assert counts["Rot"] == counts["Mul_PC"] == n1 + n2 - 1
        assert counts["Add_CC"] == n1 + n2 - 2 and counts["Add_PC"] == 1
        assert level == ctx.max_level - 1
    assert res["1"][1] == res["0"][1]


@pytest.mark.parametrize("n1,n2,tiles,parts", [(256, 10, 4, 2), (64, 3, 1, 1), (128, 16, 2, 3)])
def test_fc_hybrid_matches_direct_at_output_slots(n1, n2, tiles, parts, monkeypatch):
    """fc_forward_multi with offgrid_free=True (layers.fc_hybrid: padded-row
    diagonals as one lazy rotation sum + rotate-and-add, the fc1 evaluation of
    forward_bicrypto) vs the direct per-diagonal sum: same values at the output
    slots of every tile (to CKKS noise), identical reference counts and level;
    cifar3's own shape (two 256-wide blocks, 10 outputs, full 256-slot tiles)
    included."""
    from paper_2402_01296_b200.layers import fc_forward_multi

    rng = np.random.default_rng(n1 + 7 * n2 + parts)
    ctx = B.make_context(2048 if tiles * 256 <= 1024 else 4096, 3, 2.0 ** 50)
    S = ctx.slot_count
    step = 256 if tiles > 1 else 0
    xs = rng.standard_normal((parts, tiles, n1))
    Ws = [rng.standard_normal((n1, n2)) / np.sqrt(n1 * parts) for _ in range(parts)]
    kb = rng.standard_normal(n2)
    res = {}
    for hybrid in (True, False):
        rec = B.OpRecorder()
        blocks = []
        for pi in range(parts):
            slots = np.zeros(S)
            for tt in range(tiles):
                slots[tt * step:tt * step + n1] = xs[pi, tt]
            blocks.append((B.encrypt_vector(slots, ctx), Ws[pi]))
        out = fc_forward_multi(blocks, kb, ctx, rec, tiles=tiles, tile_step=step, offgrid_free=hybrid)
        dec = B.decrypt_vector(out, ctx)
        res[hybrid] = (np.stack([dec[tt * step:tt * step + n2] for tt in range(tiles)]), rec.snapshot(), out.level)
    want = sum(xs[pi] @ Ws[pi] for pi in range(parts)) + kb
    for hybrid, (got, counts, level) in res.items():
        assert np.abs(got - want).max() < 1e-8, hybrid
        assert level == ctx.max_level - 1
    assert res[True][1] == res[False][1]


@pytest.mark.parametrize("G,layout", [(8, 0), (64, 1)])
def test_cifar3_at_benchmarked_slot_set_counts(G, layout):
    """The conv paths the benchmark takes: G >= BCN_CONV_TC_MIN_G slot sets run
    the key-switch-fused conv MAC (materialize_conv -> conv_ks_mac) on the
    integer tensor cores -- mma.sync IMMA planes for G < 64, tcgen05 (UMMA,
    TMEM accumulators) for G >= 64 -- with the merged ModDown+rescale tail.
    Logits of every image vs the float64 reference_forward, counts and
    per-layer tables vs the reference's golden integers (one op set per G)."""
    import synthetic
    from paper_2402_01296_b200 import sim

    assert sim._conv_layout(G) == layout
    d, w, _, meta = _load("cifar3_cfg4")
    bundle = B.get("cifar3")
    sens, full = synthetic.cfg4_inputs(32 * G, seed=40 + G)
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    sim.reset_stats()
    res = B.forward_bicrypto(bundle.bi, (sens, full), w, ctx, strategy="bhw", group_size=32)
    assert res.logits_ct.batch == G
    assert res.recorder.snapshot() == meta["counts_bhw"]
    assert [list(x) for x in res.recorder.layer_table()] == meta["layer_table"]
    assert sim.STATS["keyswitch_lazy"] > 0 and sim.STATS["mac_launch"] > 0
    logits = res.decrypt_logits()
    assert logits.shape == (32 * G, 10)
    ref = B.reference_forward(bundle.bi, synthetic.decomposed(sens, full), w)
    _check(logits, ref)


def test_cifar3_two_full_slot_sets_match_reference_golden():
    """64 images = 2 full slot sets (32 x 16 x 16 = 8192 slots each): logits vs
    the unmodified reference's reference_forward AND its simulator, run set by
    set (tests/golden/make_golden.py::cifar3_cfg4_sets)."""
    d = np.load(os.path.join(GOLD, "cifar3_cfg4_sets.npz"))
    meta = json.loads(str(d["meta"]))
    w = TensorArchive({k[3:]: d[k] for k in d.files if k.startswith("w::")})
    bundle = B.get("cifar3")
    ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
    res = B.forward_bicrypto(bundle.bi, (d["sens"], d["full"]), w, ctx, strategy="bhw", group_size=32)
    assert res.recorder.snapshot() == meta["counts_bhw"]
    logits = res.decrypt_logits()
    _check(logits, d["logits_ref"])
    _check(logits, d["logits_sim"], tol=1e-6)


def _shard_worker(rank, world, port, n_sets, out_q):
    """One rank of the sharded config-4/5 forward: its contiguous slot sets,
    keys regenerated from the shared seed, logits ciphertexts gathered to
    rank 0 (gloo here: CPU copies) and decrypted there."""
    import torch
    import torch.distributed as dist

    import synthetic
    from paper_2402_01296_b200.shard import gather_to_root, shard_range

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        d, w, _, meta = _load("cifar3_cfg4")
        bundle = B.get("cifar3")
        ctx = B.make_context(1 << 14, B.required_levels(bundle) + 1, 2.0 ** 50)
        sets = shard_range(n_sets, rank, world)
        sens, full = synthetic.cfg4_set_inputs(sets, seed=77)
        res = B.forward_bicrypto(bundle.bi, (sens, full), w, ctx, strategy="bhw", group_size=32)
        assert res.recorder.snapshot() == meta["counts_bhw"]
        data = res.logits_ct.data
        c1_head = data[0, 1, 0, :64].cpu().numpy()
        got = gather_to_root(data.cpu(), n_sets)
        c1s = [None] * world
        dist.all_gather_object(c1s, c1_head)
        if rank == 0:
            slots = ctx.engine.decrypt(got.cuda(), res.logits_ct.level, res.logits_ct.scale).cpu().numpy()
            idx = np.arange(32)[:, None] * res.tile_step + np.arange(10)[None, :]
            out_q.put((slots[:, idx].reshape(-1, 10), c1s))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_forward_two_ranks_gather_matches_reference():
    """Two ranks (processes) on one GPU, each with its own shard of 4 slot sets
    (128 images): the gathered, rank-0-decrypted logits equal the reference
    for every image, and the ranks' ciphertexts carry distinct encryption
    randomness (Philox ids partitioned by rank)."""
    import socket

    import torch.multiprocessing as mp

    import synthetic

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n_sets = 4
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    ps = [ctxm.Process(target=_shard_worker, args=(r, 2, port, n_sets, q)) for r in range(2)]
    for p in ps:
        p.start()
    logits, c1s = q.get(timeout=600)
    for p in ps:
        p.join(timeout=300)
        assert p.exitcode == 0
    d, w, _, _ = _load("cifar3_cfg4")
    sens, full = synthetic.cfg4_set_inputs(range(n_sets), seed=77)
    ref = B.reference_forward(B.get("cifar3").bi, synthetic.decomposed(sens, full), w)
    assert logits.shape == (32 * n_sets, 10)
    _check(logits, ref)
    assert not np.array_equal(c1s[0], c1s[1])


def test_batched_square_is_bit_identical_to_per_channel_calls(monkeypatch):
    """sim.he_square_many (single-image path: the channels of a square layer as ONE
    Mul_CC call on the stacked batch) returns every channel's ciphertext bit for bit
    as its own he_mul(c, c) does, with the same counts."""
    import torch
    from paper_2402_01296_b200.sim import OpRecorder, encrypt_vector, he_mul, he_square_many

    ctx = B.make_context(8192, 4, 2.0 ** 50)
    rng = np.random.default_rng(2)
    cts = [encrypt_vector(rng.standard_normal(ctx.slot_count) * 0.5, ctx) for _ in range(5)]
    rec_a, rec_b = OpRecorder(), OpRecorder()
    got = he_square_many(cts, rec_a)
    want = [he_mul(c, c, rec_b) for c in cts]
    assert rec_a.counters == rec_b.counters and rec_a.counters["Mul_CC"] == 5
    for g, w in zip(got, want):
        assert g.level == w.level and g.scale == w.scale
        assert torch.equal(g.data, w.data)
    monkeypatch.setenv("BCN_BATCH_SQUARE", "0")
    for g, w in zip(he_square_many(cts, OpRecorder()), want):
        assert torch.equal(g.data, w.data)
