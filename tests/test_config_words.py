"""The harness host encoder (bench.py's and the tests' input path) produces
the reference encoder's words exactly, on the BASELINE.json config shapes
(tests/config_cases.py, encoded by oracle/_ref), so GPU results on
harness-encoded inputs are results on the reference's encoding."""
import numpy as np
import pytest

import harness as H
from tests import config_cases as CC


@pytest.fixture(scope="module")
def cases(ref):
    return CC.all_cases(ref)


def test_harness_words_equal_reference_at_every_config(cases):
    for c in cases:
        vals = c["values"]
        m = vals.shape[0]
        offs = np.arange(m, dtype=np.uint64) * CC.N
        counts = np.full(m, CC.N, dtype=np.uint32)
        e = H.encode_chunks(c["name"], vals.reshape(-1), offs, counts, allow_wrap=c["wrap"],
                            raw=c["raw"])
        assert np.array_equal(e.table["n_words"], c["table"]["n_words"]), c["label"]
        for t, r in zip(e.table, c["table"]):
            a = e.words[int(t["word_off"]):int(t["word_off"]) + int(t["n_words"])]
            b = c["words"][int(r["word_off"]):int(r["word_off"]) + int(r["n_words"])]
            assert np.array_equal(a, b), (c["label"], c["name"])


def test_reference_decodes_its_encoding_to_the_input(cases):
    for c in cases:
        assert np.array_equal(c["ref_out"], c["values"].reshape(-1)), (c["label"], c["name"])
