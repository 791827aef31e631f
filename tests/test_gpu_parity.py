"""GPU path (libcszi through the public API / C-ABI) vs the oracle and the
reference's golden archives: bit-exact archives and decompressed bytes."""
import numpy as np
import pytest

import paper_2312_05492_b200 as P
from conftest import KINDS, affine_field, constant_field, noisy_field, smooth_field
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def meta(golden):
    for m in golden["meta"]:
        i, j, mode, eb, p2, kind, shape = str(m).split("|")
        yield int(i), int(j), mode, float(eb), bool(int(p2)), kind


def test_golden_archives_bit_exact(golden):
    for i, j, mode, eb, p2, kind in meta(golden):
        data = golden[f"in_{i}"]
        g = P.Grid(P.Dims(data.shape), data)
        blob = P.compress(g, eb, mode=mode, pass2=p2)
        assert blob == golden[f"arc_{i}_{j}"].tobytes(), (i, j, mode, eb, kind, data.shape)


def test_golden_decompression_bit_exact(golden):
    for i, j, mode, eb, p2, kind in meta(golden):
        back = P.decompress(golden[f"arc_{i}_{j}"].tobytes())
        assert back.data.tobytes() == golden[f"dec_{i}_{j}"].tobytes(), (i, j)


def test_golden_sinusoid64_and_overrides(golden):
    s = O.sinusoid_64()
    g = P.Grid(P.Dims(s.shape), s)
    for eb, p2 in ((1e-3, True), (1e-2, True), (1e-4, True), (1e-3, False)):
        assert P.compress(g, eb, pass2=p2) == golden[f"s64_{eb:g}_{int(p2)}"].tobytes()
    d = golden["ovr_in"]
    g = P.Grid(P.Dims(d.shape), d)
    assert P.compress(g, 1e-3, alpha=1.25, variants=(1, 0, 1), dim_order=(2, 0, 1)) == \
        golden["ovr_arc_0"].tobytes()
    assert P.compress(g, 1e-4, quant_radius=64) == golden["ovr_arc_1"].tobytes()
    assert P.compress(g, 1e-3, mode="abs", quant_radius=3) == golden["ovr_arc_2"].tobytes()


@pytest.mark.parametrize("rank", [1, 2, 3])
def test_random_fields_vs_oracle(rank):
    rng = np.random.default_rng(1000 + rank)
    for i in range(16):
        hi = {1: 3000, 2: 90, 3: 40}[rank]
        shape = tuple(int(rng.integers(1, hi)) for _ in range(rank))
        data = KINDS[i % 4](rng, shape)
        g = P.Grid(P.Dims(shape), data)
        for mode, eb, p2 in (("rel", 1e-3, True), ("abs", 3e-2, True), ("rel", 1e-5, False),
                             ("rel", 0.3, True)):
            blob = P.compress(g, eb, mode=mode, pass2=p2)
            ref = O.compress(data, eb, mode=mode, pass2=p2)
            assert blob == ref, (shape, mode, eb)
            assert P.decompress(blob).data.tobytes() == O.decompress(ref).tobytes()


def test_irregular_3d_shapes_vs_oracle():
    rng = np.random.default_rng(11)
    for shape in ((53, 47, 71), (33, 69, 69), (17, 65, 129), (9, 8, 33), (8, 16, 32),
                  (16, 17, 64), (1, 1, 1), (2, 2, 2), (70, 3, 5)):
        data = smooth_field(rng, shape)
        g = P.Grid(P.Dims(shape), data)
        for eb in (1e-2, 1e-4):
            blob = P.compress(g, eb)
            assert blob == O.compress(data, eb), shape
            assert P.decompress(blob).data.tobytes() == O.decompress(blob).tobytes()


def test_exact_fit_edge_tiles_vs_oracle():
    """Edge tiles whose axes end exactly on the tile boundary (z, y = 8,
    x = 32: tile3i.cuh fit_mask) run the interior walks with the end cases;
    every fit mask, pass order and cubic variant, with outliers and exact
    redos (noisy data at tight bounds) and the closing anchors they keep."""
    rng = np.random.default_rng(23)
    shapes = ((8, 8, 32), (16, 16, 64), (8, 24, 96), (24, 8, 33), (9, 16, 64), (16, 9, 32),
              (8, 8, 65), (17, 16, 64))
    for si, shape in enumerate(shapes):
        for kind in (smooth_field, noisy_field):
            data = kind(rng, shape)
            g = P.Grid(P.Dims(shape), data)
            opts = [dict(eb=1e-3), dict(eb=1e-5), dict(eb=3e-2, mode="abs", quant_radius=4)]
            order = [(0, 1, 2), (2, 0, 1), (1, 2, 0), (2, 1, 0)][si % 4]
            variants = [(1, 0, 1), (0, 1, 0)][si % 2]
            opts.append(dict(eb=1e-4, dim_order=order, variants=variants, alpha=1.25))
            for o in opts:
                o = dict(o)
                eb = o.pop("eb")
                blob = P.compress(g, eb, **o)
                assert blob == O.compress(data, eb, **o), (shape, kind.__name__, eb, o)
                assert P.decompress(blob).data.tobytes() == O.decompress(blob).tobytes(), \
                    (shape, kind.__name__, eb, o)


def test_exact_fit_tiles_match_generic_walks():
    """The same fields through the generic (exact) walks: byte-identical
    archives at sizes the oracle would take minutes on."""
    rng = np.random.default_rng(29)
    for shape in ((64, 48, 128), (40, 72, 96)):
        for kind in (smooth_field, noisy_field):
            data = kind(rng, shape)
            g = P.Grid(P.Dims(shape), data)
            for eb in (1e-3, 1e-5):
                a = P.compress_device(g, eb).to_bytes()
                b = P.compress_device(g, eb, exact=True).to_bytes()
                assert a == b, (shape, kind.__name__, eb)


def test_compress_predict_matches_oracle():
    rng = np.random.default_rng(5)
    for shape in ((40, 33, 47), (64, 64), (5000,)):
        data = noisy_field(rng, shape)
        for mode, eb in (("rel", 1e-3), ("rel", 1e-5)):
            cfg = O.select_config(data, mode, eb)
            codes, is_out, rec = O.predict(data, cfg)
            pc = P.PredictorConfig(P.ChunkLayout(cfg.stride, cfg.rank, cfg.tiles), cfg.alpha,
                                   cfg.variants, cfg.dim_order, cfg.eb_abs)
            g = P.Grid(P.Dims(shape), data)
            qf = P.compress_predict(g, pc)
            assert np.array_equal(qf.codes, codes)
            oidx = np.nonzero(is_out)[0]
            assert [i for i, _ in qf.outliers] == oidx.tolist()
            back = P.decompress_predict(qf, pc, P.Dims(shape))
            assert back.data.tobytes() == rec.tobytes()


def test_fast_quantizer_equals_exact_division():
    """The reciprocal fast path must reproduce t = (o - pred) / e2 exactly."""
    from paper_2312_05492_b200.predictor import _run_predict

    rng = np.random.default_rng(17)
    for shape, kind in (((48, 40, 64), noisy_field), ((33, 70, 45), smooth_field)):
        data = kind(rng, shape)
        g = P.Grid(P.Dims(shape), data)
        for eb in (1e-1, 1e-3, 3.3e-4, 1e-5, 7.77e-6):
            cfg = O.select_config(data, "rel", eb)
            pc = P.PredictorConfig(P.default_layout(3), cfg.alpha, cfg.variants, cfg.dim_order,
                                   cfg.eb_abs)
            a, ha, _, _ = _run_predict(g, pc, exact=False)
            b, hb, _, _ = _run_predict(g, pc, exact=True)
            assert bool((a == b).all()) and bool((ha == hb).all()), eb


def test_device_resident_round_trip():
    import torch

    rng = np.random.default_rng(2)
    data = smooth_field(rng, (37, 41, 96))
    x = torch.from_numpy(data).cuda()
    g = P.Grid(P.Dims(data.shape), x)
    assert g.is_device
    arch = P.compress_device(g, 1e-3)
    assert arch.to_bytes() == O.compress(data, 1e-3)
    y = P.decompress_device(arch)
    assert y.is_device
    assert y.data.tobytes() == O.decompress(arch.to_bytes()).tobytes()
    lo, hi, rng_ = P.value_range(g)
    assert (lo, hi) == (float(data.min()), float(data.max()))


def test_constant_and_affine_fields():
    rng = np.random.default_rng(5)
    g = P.Grid(P.Dims((64, 64, 64)), constant_field(rng, (64, 64, 64)))
    blob = P.compress(g, 1e-3)
    assert 8.0 * len(blob) / g.dims.count < 1.0
    assert P.decompress(blob) == g
    for shape in ((513,), (17, 33), (9, 17, 33), (65, 49)):
        data = affine_field(rng, shape)
        cfg = O.select_config(data, "rel", 1e-3)
        pc = P.PredictorConfig(P.ChunkLayout(cfg.stride, cfg.rank, cfg.tiles), cfg.alpha,
                               cfg.variants, cfg.dim_order, cfg.eb_abs)
        qf = P.compress_predict(P.Grid(P.Dims(shape), data), pc)
        assert not qf.codes.any() and not qf.outliers


def test_thread_count_never_changes_bytes():
    rng = np.random.default_rng(77)
    g = P.Grid(P.Dims((33, 29, 31)), smooth_field(rng, (33, 29, 31)))
    blobs = [P.compress(g, 1e-3, threads=t) for t in (1, 2, 5)]
    assert blobs[0] == blobs[1] == blobs[2]


def test_error_bound_battery():
    rng = np.random.default_rng(2024)
    for i in range(60):
        rank = i % 3 + 1
        shape = tuple(int(rng.integers(5, 60)) for _ in range(rank))
        g = P.Grid(P.Dims(shape), KINDS[i % 4](rng, shape))
        for mode in ("abs", "rel"):
            for eb in (1e-1, 1e-3, 1e-5):
                blob = P.compress(g, eb, mode=mode)
                out = P.decompress(blob)
                rep = P.verify_error_bound(g, out, P.parse_archive(blob).eb_abs)
                assert rep.ok, (shape, mode, eb, rep)
