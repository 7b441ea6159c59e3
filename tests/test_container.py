"""INTZPK01 container ingest (container.h:14-26, container.cpp:93-169) against
the reference's own reader and writer (compiled from source, oracle/_ref).

CPU tests: for containers written by the reference, our in-place index must
yield exactly the chunks container_read_encoded returns; for corrupted
containers our status must be the reference's first CorruptError (same
what() text).  The GPU test decodes whole containers through
izg_container_decode_host.
"""
import zlib

import numpy as np
import pytest

import paper_1209_2137_b200 as P
from paper_1209_2137_b200 import container as CT
from tests.helpers import REF_NAMES, random_sorted


def arrays_for(seed, sizes=(0, 1, 127, 128, 300, 2048, 65536, 65537, 140000)):
    rng = np.random.default_rng(seed)
    return [random_sorted(rng, n, int(rng.choice([3, 1000, 1 << 20]))) for n in sizes]


def chunks_of_container(c: CT.Container):
    t, w = c.encoded.table, c.encoded.words
    out = []
    for a in range(len(c.array_chunk0) - 1):
        out.append([(int(x["n"]), w[int(x["word_off"]):int(x["word_off"]) + int(x["n_words"])])
                    for x in t[c.array_chunk0[a]:c.array_chunk0[a + 1]]])
    return out


@pytest.mark.parametrize("name", REF_NAMES)
def test_index_matches_reference_reader(ref, name):
    arrays = arrays_for(zlib.crc32(name.encode()) % 1000)
    data = ref.container_write_encoded(name, arrays)
    rname, rarrays = ref.container_read_encoded(data)
    c = CT.read_container(data)
    assert c.codec_name == rname == name
    ours = chunks_of_container(c)
    assert len(ours) == len(rarrays) == len(arrays)
    for a, (x, y) in enumerate(zip(ours, rarrays)):
        assert len(x) == len(y), a
        for (n0, p0), (n1, p1) in zip(x, y):
            assert n0 == n1 and np.array_equal(p0, p1), a
    # array offsets: arrays back to back
    assert list(np.diff(c.array_offsets)) == [len(a) for a in arrays]
    # the placement satisfies izg_decode's contract (16-byte rows inside words)
    t = c.encoded.table
    assert int((t["word_off"] + t["n_words"]).max()) <= len(c.encoded.words) - 3


def test_raw_container_matches_reference(ref):
    arrays = arrays_for(5, sizes=(0, 1, 5, 1000))
    data = ref.container_write_raw(arrays)
    got = CT.read_raw_container(data)
    want = ref.container_read_raw(data)
    assert len(got) == len(want) == len(arrays)
    for g, w, a in zip(got, want, arrays):
        assert np.array_equal(g, w) and np.array_equal(g, a)
    # reading RAW as encoded (and vice versa) fails like the reference
    for fn, wrong in ((CT.read_container, data),
                      (CT.read_raw_container, ref.container_write_encoded("simdbp128", arrays))):
        with pytest.raises(P.CorruptError) as e:
            fn(wrong)
        assert str(e.value).startswith("container: expected")


def ref_status(ref, data, raw=False):
    from oracle.pyoracle import RefError

    try:
        (ref.container_read_raw if raw else ref.container_read_encoded)(data)
        return None
    except RefError as e:
        assert e.code == 1, e.what  # CorruptError only
        return e.what


def our_status(data, raw=False):
    try:
        CT.scan_container(data, raw=raw)
        return None
    except P.CorruptError as e:
        return str(e)


def mutants(rng, data: bytes):
    b = bytearray(data)
    out = [bytes(b[:k]) for k in range(0, min(len(b), 64))]          # every early cut
    out += [bytes(b[:k]) for k in rng.integers(0, len(b), size=40)]   # later cuts
    body = 8 + 4 + int.from_bytes(b[8:12], "little") + 4

    def put(off, v):
        m = bytearray(b)
        if off + 4 <= len(m):
            m[off:off + 4] = (v & 0xFFFFFFFF).to_bytes(4, "little")
        out.append(bytes(m))

    for v in (0, 257, 1 << 31, 3):
        put(8, v)                                                # name length
    m = bytearray(b); m[3] ^= 1; out.append(bytes(m))           # magic
    n_arrays = int.from_bytes(b[body - 4:body], "little")
    for d in (-1, 1, 1000):
        put(body - 4, n_arrays + d)
    # walk the array records and mutate their fields and chunk records
    pos = body
    for _ in range(n_arrays):
        ol = int.from_bytes(b[pos:pos + 4], "little")
        wc = int.from_bytes(b[pos + 4:pos + 8], "little")
        for d in (-1, 1):
            put(pos, ol + d)
            put(pos + 4, wc + d)
        q = pos + 8
        end = q + 4 * wc
        while q + 8 <= end:
            n = int.from_bytes(b[q:q + 4], "little")
            nw = int.from_bytes(b[q + 4:q + 8], "little")
            for v in (0, 65537, n + 1, n - 1):
                put(q, v)
            for v in (nw + 1, nw + 1000, 1 << 31):
                put(q + 4, v)
            q += 8 + 4 * nw
        pos = end
    return out


@pytest.mark.parametrize("name", ["simdbp128-s4", "simdfastpfor"])
def test_corrupt_containers_match_reference(ref, name):
    rng = np.random.default_rng(11)
    arrays = arrays_for(3, sizes=(0, 5, 300, 70000))
    data = ref.container_write_encoded(name, arrays)
    ms = mutants(rng, data)
    seen = set()
    for i, m in enumerate(ms):
        want, got = ref_status(ref, m), our_status(m)
        assert got == want, (i, len(m), got, want)
        seen.add(got)
        if want is None:  # accepted: the index must agree with the reference too
            _, rarrays = ref.container_read_encoded(m)
            ours = chunks_of_container(CT.read_container(m))
            assert [[(n, p.tolist()) for n, p in a] for a in ours] == \
                   [[(n, p.tolist()) for n, p in a] for a in rarrays]
    # the mutants reach every encoded-container throw site
    assert {"container: truncated", "container: bad magic", "container: bad codec name length",
            "container: truncated payload", "container: truncated chunk record",
            "container: bad chunk length", "container: bad chunk word count",
            "container: array length mismatch"} <= seen, seen


def test_corrupt_raw_containers_match_reference(ref):
    rng = np.random.default_rng(12)
    data = ref.container_write_raw(arrays_for(4, sizes=(0, 3, 50)))
    seen = set()
    for m in mutants(rng, data)[:120]:
        want = ref_status(ref, m, raw=True)
        got = our_status(m, raw=True)
        if want and want.startswith("container: expected RAW data, found codec"):
            assert got == "container: expected RAW data, found codec"
        else:
            assert got == want, (len(m), got, want)
        seen.add(got)
    assert "container: RAW word count mismatch" in seen


def test_golden_container_fixture():
    """A committed container written by the reference (tests/golden/
    make_golden.py): indexes to the recorded chunk table."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.npz"))
    if "container_bytes" not in g:
        pytest.skip("fixture predates containers")
    c = CT.read_container(g["container_bytes"].tobytes())
    assert c.codec_name == "simdbp128-s4"
    t = c.encoded.table
    assert np.array_equal(t["n"], g["container_n"])
    assert np.array_equal(t["n_words"], g["container_n_words"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", REF_NAMES)
def test_decode_container_on_gpu(cuda, ref, name):
    arrays = arrays_for(zlib.crc32(name.encode()) % 777)
    data = ref.container_write_encoded(name, arrays)
    values, offs = CT.decode_container(data)
    assert np.array_equal(values, np.concatenate(arrays))
    assert list(np.diff(offs)) == [len(a) for a in arrays]
    # a corrupt chunk inside a valid container raises the chunk's status
    c = CT.read_container(data)
    k = int(np.argmax(c.encoded.table["n_words"]))
    at = int(c.encoded.table["word_off"][k])
    b = bytearray(data)
    o = 8 + 4 + len(name) + 4 + 4 * at
    b[o:o + 4] = (0xFFFFFFFF).to_bytes(4, "little")
    with pytest.raises((P.CorruptError, ValueError)):
        CT.decode_container(bytes(b))


@pytest.mark.gpu
def test_golden_container_decodes_on_gpu(cuda):
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.npz"))
    values, offs = CT.decode_container(g["container_bytes"].tobytes())
    assert np.array_equal(values, g["container_values"])
