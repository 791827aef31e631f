"""Stage-level GPU parity: histogram, codebook, Huffman encode/decode, pass-2,
profiling, anchors — each against the oracle and the reference's known answers."""
import numpy as np
import pytest

import paper_2312_05492_b200 as P
from conftest import noisy_field, smooth_field
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_pass2_known_answers_and_random():
    assert P.pass2_encode(b"\x00" * 5) == b"\x84"
    assert P.pass2_encode(b"AB") == b"\x01AB"
    assert P.pass2_encode(b"") == b""
    assert P.pass2_encode(b"\x00") == b"\x00\x00"
    assert P.pass2_encode(b"A\x00B") == b"\x02A\x00B"
    assert P.pass2_encode(b"\x00" * 300) == b"\xff\xff" + bytes([127 + 44])
    data = bytes(range(1, 256)) * 2
    assert P.pass2_encode(data)[0] == 127
    with pytest.raises(P.Corrupt):
        P.pass2_decode(b"\x05AB")
    with pytest.raises(P.Corrupt):
        P.pass2_encode(b"abc", codec=250)
    rng = np.random.default_rng(4)
    for n in (1, 2, 3, 127, 128, 129, 4095, 4096, 4097, 20000, 300000):
        for p in (0.0, 0.5, 0.9, 1.0):
            raw = rng.integers(1, 256, n).astype(np.uint8)
            raw[rng.random(n) < p] = 0
            data = raw.tobytes()
            enc = P.pass2_encode(data)
            assert enc == O.pass2_encode(data), (n, p)
            assert len(enc) <= len(data) + len(data) // 128 + 1
            assert P.pass2_decode(enc) == data


def test_pass2_runs_across_tiles():
    """Zero runs / literal stretches of random lengths straddling the 4 KiB
    encoder tiles and the 128-byte chunk limit, vs the oracle."""
    rng = np.random.default_rng(11)
    for mean_run, mean_lit in ((3, 2), (150, 40), (700, 300), (5000, 129)):
        parts = []
        total = 0
        while total < 60000:
            r = int(rng.geometric(1.0 / mean_run))
            lit = rng.integers(1, 256, int(rng.geometric(1.0 / mean_lit))).astype(np.uint8)
            lit[rng.random(lit.size) < 0.1] = 0  # isolated zeros stay literal
            parts += [np.zeros(r, np.uint8), lit]
            total += r + lit.size
        data = np.concatenate(parts).tobytes()
        for cut in (len(data), 4096 * 3 + 1, 4096 * 2, 4095, 128 * 7 + 2):
            d = data[:cut]
            enc = P.pass2_encode(d)
            assert enc == O.pass2_encode(d), (mean_run, mean_lit, cut)
            assert P.pass2_decode(enc) == d


def test_pass2_registry():
    P.register_pass2_codec(9, lambda d: bytes(b ^ 0x55 for b in d),
                           lambda d: bytes(b ^ 0x55 for b in d))
    payload = b"\x00\x00hello"
    assert P.pass2_decode(P.pass2_encode(payload, codec=9), codec=9) == payload
    with pytest.raises(ValueError):
        P.register_pass2_codec(0, None, None)
    rng = np.random.default_rng(1)
    g = P.Grid(P.Dims((20, 30)), smooth_field(rng, (20, 30)))
    blob = P.compress(g, 1e-3, pass2_codec=9)
    assert P.parse_archive(blob).pass2_codec == 9
    assert P.decompress(blob) == P.decompress(P.compress(g, 1e-3))


def test_histogram_codebook_encode_decode_vs_oracle():
    rng = np.random.default_rng(7)
    for R, gen in ((512, lambda n: rng.integers(-20, 21, n)), (32, lambda n: rng.integers(-3, 4, n)),
                   (512, lambda n: np.round(rng.laplace(0, 30, n)).clip(-511, 511)),
                   (8, lambda n: rng.integers(0, 8, n) - 4), (4, lambda n: np.zeros(n))):
        for n in (1, 10, 4095, 4096, 4097, 100000):
            codes = gen(n).astype(np.int32)
            h = P.build_histogram(codes, R)
            assert np.array_equal(h.counts, O.histogram(codes, R))
            cb = P.build_codebook(h)
            ocb = O.canonical(O.code_lengths(O.histogram(codes, R)))
            assert np.array_equal(cb.code_lengths, ocb.lengths)
            assert np.array_equal(cb.words, ocb.words)
            assert np.array_equal(cb.first_code, ocb.first_code)
            assert np.array_equal(cb.sorted_symbols, ocb.sorted_symbols)
            stream, bits = P.huffman_encode(codes, cb)
            ostream, obits = O.huffman_encode(codes, ocb, R)
            assert (stream, bits) == (ostream, obits)
            assert np.array_equal(P.huffman_decode(stream, cb, n), codes)


def test_huffman_known_answers_and_errors():
    book = P.build_codebook(P.build_histogram(np.asarray([-3] * 3 + [-2, -1], np.int32), 4))
    assert {s: int(l) for s, l in enumerate(book.code_lengths) if l} == {1: 1, 2: 2, 3: 2}
    assert [int(book.words[s]) for s in (1, 2, 3)] == [0b0, 0b10, 0b11]
    book = P.Codebook.from_lengths(np.asarray([1, 2, 2, 0], np.uint8))
    stream, bits = P.huffman_encode(np.asarray([-2, -2, -1], np.int32), book)
    assert bits == 4 and stream[:1] == b"\x20"
    one = P.build_codebook(P.build_histogram(np.zeros(10, np.int32), 4))
    assert one.code_lengths[4] == 1
    s, b = P.huffman_encode(np.zeros(10, np.int32), one)
    assert b == 10 and P.huffman_decode(s, one, 10).tolist() == [0] * 10
    with pytest.raises(P.EmptyHistogram):
        P.build_codebook(P.build_histogram(np.zeros(0, np.int32), 2))
    with pytest.raises(P.OutOfRange):
        P.build_histogram(np.asarray([2], np.int32), 2)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    counts = np.zeros(128, np.int64)
    counts[:40] = fib
    with pytest.raises(P.LengthOverflow):
        P.build_codebook(P.Histogram(counts))
    book = P.build_codebook(P.build_histogram(np.asarray([0, 1], np.int32), 2))
    with pytest.raises(P.UnknownSymbol):
        P.huffman_encode(np.asarray([-2], np.int32), book)
    codes = np.asarray([0, 1, -1, 0, 1, 1, 0, -1] * 8, np.int32)
    book = P.build_codebook(P.build_histogram(codes, 2))
    stream, bits = P.huffman_encode(codes, book)
    with pytest.raises(P.TruncatedStream):
        P.huffman_decode(stream[: max(1, (bits // 8) // 2)], book, codes.size)


def test_decode_without_resynchronisation():
    """Equal code lengths never self-synchronise: the exact table fallback."""
    rng = np.random.default_rng(9)
    for k in (8, 16, 3, 5):
        codes = rng.integers(0, k, 200000).astype(np.int32) - k // 2
        book = P.build_codebook(P.build_histogram(codes, 16))
        stream, _ = P.huffman_encode(codes, book)
        assert np.array_equal(P.huffman_decode(stream, book, codes.size), codes)


def test_profile_and_gather_anchors():
    rng = np.random.default_rng(3)
    for shape in ((64, 64, 64), (30, 7, 50), (6, 100), (2000,), (9, 9, 9)):
        data = noisy_field(rng, shape)
        g = P.Grid(P.Dims(shape), data)
        st = P.profile_samples(g)
        lo, hi, rng_, err, cnt = O.profile(data)
        assert (st.value_min, st.value_max, st.value_range) == (lo, hi, rng_)
        assert np.array_equal(st.err_sum, err) and np.array_equal(st.sample_count, cnt)
        anchors = P.gather_anchors(g, 8)
        idx = O.anchor_flat_indices(shape, 8)
        assert [i for i, _ in anchors] == idx.tolist()
        assert [v for _, v in anchors] == data.ravel()[idx].tolist()


def test_pass2_decode_chunk_boundaries():
    """Encoded streams built control by control so literal payloads (up to
    128 bytes) and zero-run controls straddle the decoder's 256-byte chunks
    at every offset: the transfer tables' spill entries (0..128), a chunk
    whose first bytes are the previous chunk's payload, streams ending inside
    a chunk, and an overrun in the last chunk -- vs the oracle."""
    rng = np.random.default_rng(23)
    for trial in range(60):
        out = bytearray()
        target = int(rng.integers(1, 3000))
        while len(out) < target:
            if rng.random() < 0.5:
                k = int(rng.integers(1, 129))
                out.append(k - 1)
                out += bytes(rng.integers(0, 256, k).astype(np.uint8))
            else:
                out.append(int(rng.integers(128, 256)))
        enc = bytes(out)
        assert P.pass2_decode(enc) == O.pass2_decode(enc), trial
    # a literal header at every offset of the chunk's last 130 bytes
    for off in range(256 - 130, 257):
        body = bytes([0xFF]) * off + bytes([127]) + bytes(rng.integers(0, 256, 128).astype(np.uint8))
        enc = body + bytes([0x80, 5, 1, 2, 3, 4, 5, 6])
        assert P.pass2_decode(enc) == O.pass2_decode(enc), off
        with pytest.raises(P.Corrupt):
            P.pass2_decode(body[:-1])  # the literal overruns the stream
