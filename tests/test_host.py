"""Host-side logic of the drop-in API that needs no GPU: recorder algebra,
layouts, catalog/depth budgets vs the reference's pinned numbers, parameter
checks, archives, the numpy clear forward vs the reference's golden logits,
C-ABI library exports, and the gloo (world_size 2) sharding path."""

import json
import os
import re
import socket

import numpy as np
import pytest

import paper_2402_01296_b200 as B
from paper_2402_01296_b200 import catalog
from paper_2402_01296_b200.archive import TensorArchive, write_archive
from paper_2402_01296_b200.errors import ArchiveError, CapacityError, ParameterError, UsageError
from paper_2402_01296_b200.network import DecomposedInput

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _gold(name):
    d = np.load(os.path.join(GOLD, name + ".npz"))
    w = TensorArchive({k[3:]: d[k] for k in d.files if k.startswith("w::")})
    dec = [DecomposedInput(s, f, (0, 0, 0, 0)) for s, f in zip(d["sens"], d["full"])]
    return d, w, dec, json.loads(str(d["meta"]))


# ---------------------------------------------------------------- recorder
def test_recorder_layers_sum_to_totals_and_nest():
    rec = B.OpRecorder()
    with rec.layer("outer"):
        rec.bump("Add_PC")
        with rec.layer("inner"):
            rec.bump("Add_CC", 2)
    rec.bump("Rot")
    table = dict(rec.layer_table())
    assert table["outer"]["Add_PC"] == 1 and table["outer"]["Add_CC"] == 0
    assert table["inner"]["Add_CC"] == 2
    assert table["(unscoped)"]["Rot"] == 1
    for k, v in rec.counters.items():
        assert sum(d[k] for _, d in rec.layer_table()) == v
    assert rec.current_layer is None


def test_recorder_merge_equals_sequential():
    seq, workers = B.OpRecorder(), []
    for i in range(4):
        with seq.layer(f"ch{i}"):
            seq.bump("Mul_PC", i + 1)
        w = B.OpRecorder()
        with w.layer(f"ch{i}"):
            w.bump("Mul_PC", i + 1)
        workers.append(w)
    merged = B.OpRecorder()
    for w in workers:
        merged.merge(w)
    assert merged.counters == seq.counters and merged.layer_table() == seq.layer_table()


# ---------------------------------------------------------------- context
def test_make_context_checks_match_reference():
    assert B.make_context(1 << 14, 10, 2.0 ** 30).slot_count == 8192
    assert B.make_context(8, 1, 1.0).slot_count == 4
    for bad in (7, 12, 100, 0, 4):
        with pytest.raises(ParameterError):
            B.make_context(bad, 1, 1.0)
    with pytest.raises(ParameterError):
        B.make_context(8, 0, 1.0)
    with pytest.raises(ParameterError):
        B.make_context(8, 1, -1.0)
    with pytest.raises(ParameterError):
        B.make_context(8, 1, 1.0, scheme="RSA")
    ctx = B.make_context(1 << 14, 10, 2.0 ** 30, scheme="CKKS")
    assert ctx.latency_table["Add_PC"] == 0.039 and ctx.latency_table["Rot"] == ctx.latency_table["Mul_PC"]


def test_context_chain_follows_depth_budget():
    bundle = B.get("cnn3")
    ctx = B.make_context(**B.default_context_params(bundle))
    assert ctx.max_level == 10 and len(ctx.he.q) == 11
    assert all(q % (2 * ctx.poly_degree) == 1 for q in ctx.he.q + ctx.he.p)
    assert ctx.he.K == -(-(ctx.max_level + 1) // ctx.he.dnum)


# ---------------------------------------------------------------- packing
def test_layout_capacity_and_indices():
    lay = B.PackLayout("bhw", 2, 4, 4, 3, 64)
    assert lay.slots_needed() == 32 and lay.ciphertext_count() == 3
    assert B.slot_index(1, 2, 3, lay) == 16 + 8 + 3
    with pytest.raises(CapacityError):
        B.PackLayout("bhw", 8192, 1, 2, 1, 8192)
    with pytest.raises(UsageError):
        B.PackLayout("zz", 1, 1, 1, 1, 8)
    with pytest.raises(IndexError):
        B.slot_index(2, 0, 0, lay)


def test_slot_rows_follow_index_rule():
    from paper_2402_01296_b200.packing import slot_rows

    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 4, 5))
    for strat in ("bhw", "hw", "batch"):
        lay = B.PackLayout(strat, 2, 4, 5, 3, 64)
        rows = slot_rows(x, lay)
        assert rows.shape[0] == lay.ciphertext_count()
        if strat == "bhw":
            assert rows[1, B.slot_index(1, 2, 3, lay)] == x[1, 1, 2, 3]
        elif strat == "hw":
            assert rows[1 * 3 + 2, B.slot_index(1, 2, 3, lay)] == x[1, 2, 2, 3]
        else:
            assert rows[1 * 20 + 2 * 5 + 3, B.slot_index(1, 2, 3, lay)] == x[1, 1, 2, 3]


# ---------------------------------------------------------------- catalog
@pytest.mark.parametrize("arch,n_c,n_p,head", [("cnn3", 125, 720, (100, 10)), ("cnn11", 512, 2048, (256, 10)),
                                               ("vgg16", 512, 512, (512, 10)),
                                               ("resnet18", 2048, 8192, (512, 10)),
                                               ("cifar3", 512, 2048, (20, 10))])
def test_catalog_widths(arch, n_c, n_p, head):
    sh = catalog.branch_shapes(catalog.get(arch).bi)
    assert (sh["n_c"], sh["n_p"], sh["head"]) == (n_c, n_p, head)


def test_required_levels_pins():
    d, _, _, meta = _gold("cnn3_fixture")
    bundle = catalog.get("cnn3")
    assert [catalog.required_levels(bundle.bi), catalog.required_levels(bundle.backbone)] == meta["required_levels"]
    assert catalog.required_levels(catalog.get("cifar3").bi) == 13


# ---------------------------------------------------------------- network (host parts)
def test_clear_forward_matches_reference_golden():
    for name, arch in (("cnn3_fixture", "cnn3"), ("cnn3_cfg1", "cnn3"), ("cifar3_cfg4", "cifar3"),
                      ("cifar3_cfg4_sets", "cifar3")):
        d, w, dec, _ = _gold(name)
        got = B.reference_forward(catalog.get(arch).bi, dec, w)
        assert np.abs(got - d["logits_ref"]).max() <= 1e-12 * max(1.0, np.abs(d["logits_ref"]).max())


def test_clear_backbone_matches_reference_golden():
    """reference_backbone (single-chain clear forward, network.py:585-604) ==
    the reference's logits on the golden image."""
    d = np.load(os.path.join(GOLD, "cnn3_backbone.npz"))
    from paper_2402_01296_b200.archive import TensorArchive
    w = TensorArchive({k[3:]: d[k] for k in d.files if k.startswith("w::")})
    got = B.reference_backbone(catalog.get("cnn3").backbone, d["image"][None], w)
    assert np.abs(got - d["logits_ref"]).max() <= 1e-12 * max(1.0, np.abs(d["logits_ref"]).max())


def test_decompose_and_crop_semantics():
    img = np.arange(16.0).reshape(1, 4, 4)
    d = B.decompose_input(img, noise_sigma=0.0, seed=0)
    assert d.region == (1, 1, 2, 2) and np.array_equal(d.sensitive, img[:, 1:3, 1:3])
    assert not d.plain_full[:, 1:3, 1:3].any()
    a = B.decompose_input(np.ones((3, 8, 8)), 0.1, 42)
    b = B.decompose_input(np.ones((3, 8, 8)), 0.1, 42)
    assert np.array_equal(a.plain_full, b.plain_full)
    x = np.arange(25.0).reshape(1, 5, 5)
    assert np.array_equal(B.resize_crop(x, (2, 2))[0], [[6.0, 7.0], [11.0, 12.0]])


def test_taint_check_flags_plain_layers():
    rec = B.OpRecorder()
    with rec.layer("plain.0.conv"):
        rec.bump("Mul_PC")
    with rec.layer("cipher.0.conv"):
        rec.bump("Rot")
    v = B.taint_check(catalog.get("cnn3").bi, rec)
    assert not v.passed and v.violations == ("plain.0.conv",)


def test_archive_roundtrip_and_validation(tmp_path):
    t = {"a": np.arange(6.0).reshape(2, 3), "b": np.ones(4)}
    write_archive(str(tmp_path / "w"), t, {"k": 1})
    back = TensorArchive.load(str(tmp_path / "w"))
    assert np.array_equal(back["a"], t["a"]) and back.meta == {"k": 1}
    with pytest.raises(ArchiveError):
        back["missing"]


# ---------------------------------------------------------------- C ABI
def test_library_exports_every_header_symbol():
    from paper_2402_01296_b200 import _lib

    header = open(os.path.join(ROOT, "include", "bcn.h")).read()
    declared = set(re.findall(r"\b(bcn(?:32)?_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.exported_symbols())
    lib = _lib.load()          # loads without a GPU; no compute call here
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.bcn_version() == 1


# ---------------------------------------------------------------- sharding (gloo, world 2)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_items, out_q):
    import torch
    import torch.distributed as dist

    from paper_2402_01296_b200.engine import counter_base, process_rank
    from paper_2402_01296_b200.shard import gather_to_root, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    assert process_rank() == rank                 # the engine's encryption-id base follows the job rank
    bases = [None] * world
    dist.all_gather_object(bases, counter_base(process_rank()))
    assert len(set(bases)) == world
    mine = shard_range(n_items, rank, world)
    local = torch.stack([torch.full((2, 3), float(i)) for i in mine]) if len(mine) else torch.zeros((0, 2, 3))
    got = gather_to_root(local, n_items)
    if rank == 0:
        out_q.put(got.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_items", [5, 8, 1])
def test_sharded_gather_world2_gloo(n_items):
    import torch.multiprocessing as mp

    from paper_2402_01296_b200.shard import shard_range

    assert sum(len(shard_range(n_items, r, 2)) for r in range(2)) == n_items
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n_items, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got[:, 0, 0], np.arange(n_items, dtype=float))


def test_encryption_id_ranges_are_disjoint_per_rank():
    """Philox encryption ids: rank r owns [1 + r 2^40, 1 + (r+1) 2^40)."""
    from paper_2402_01296_b200.engine import RANK_ID_SHIFT, counter_base

    assert counter_base(0) == 1
    assert counter_base(1) - counter_base(0) == 1 << RANK_ID_SHIFT
    assert len({counter_base(r) for r in range(8)}) == 8
    with pytest.raises(Exception):
        counter_base(-1)


def test_latency_table_has_the_reference_cost_model_format():
    """profiles/latency_table_b200.json (tools/latency_table.py) follows the
    BIBRANCH_LATENCY_TABLE override format of the reference's cost model
    (costs.py:22-47): {scheme: {op: ms}} with every HE op positive."""
    path = os.path.join(ROOT, "profiles", "latency_table_b200.json")
    tab = json.load(open(path))
    for scheme in ("CKKS_B200", "CKKS_B200_G128"):
        ops = tab[scheme]
        for k in ("Add_PC", "Add_CC", "Mul_PC", "Mul_CC", "Rot"):
            assert ops[k] > 0


@pytest.mark.parametrize("geom", [((28, 28), (5, 5), (2, 2), (0, 0)), ((32, 32), (3, 3), (1, 1), (1, 1)),
                                  ((32, 32), (3, 3), (2, 2), (1, 1)), ((14, 14), (5, 5), (1, 1), (0, 0))])
@pytest.mark.parametrize("tiles", [1, 4])
def test_conv_tap_patterns_vanish_off_the_output_grid(geom, tiles):
    """sim.he_mul_support_mask realises a conv layer's output-mask product as a
    level drop: valid because every tap pattern (layers._tap_pattern) is zero
    off the output grid, so the conv output's support is inside the mask."""
    from paper_2402_01296_b200.layers import SlotGrid, _grid_pattern, _tap_pattern, conv_geometry

    (h, w), k, stride, pad = geom
    S = 8192
    grid = SlotGrid(h, w, tiles=tiles, tile_step=S // tiles if tiles > 1 else 0)
    out = conv_geometry(grid, k, stride, pad)
    mask = _grid_pattern(out, S)
    for di in range(k[0]):
        for dj in range(k[1]):
            tap = _tap_pattern(grid, out, stride, pad, di, dj, S)
            assert not np.any(tap[mask == 0]), (di, dj)
