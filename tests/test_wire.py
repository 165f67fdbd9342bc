"""Wire formats against the compiled reference (oracle/_ref):
tensor JSON (tensor.cpp:132-147) byte-identical output and bit-identical reads, tensor binary
(tensor.cpp:149-186) byte-identical, layer descriptor JSON (layers.cpp:425-467) identical
round trips and the same errors.  Host-only (no device)."""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from paper_2401_03384_b200 import wire
from oracle import np_oracle as npo

SPECIAL = [0.0, -0.0, 1.0, -2.0, 0.1, 1.0 / 3.0, 1e-5, 1.5e-4, 0.001, 123456.789, 1e15, 1e16, 1.2345e20, 5e-324,
           1.7976931348623157e308, -9.87654321e-10, 2.0 ** 60, 100.0, 12345678901234567890.0]


def test_tensor_json_matches_reference_bytes(ref):
    for shape, seed in [([3, 4], 1), ([2, 3, 5], 7), ([1], 3), ([64, 33], 11)]:
        a = npo.fill_random(shape, seed)
        assert wire.tensor_to_json(a) == ref.tensor_to_json(a), shape
    s = np.array(SPECIAL)
    assert wire.tensor_to_json(s) == ref.tensor_to_json(s)
    # FP32-rounded values as the device produces them, widened to FP64 on the wire
    f = npo.fill_random([4096], 5).astype(np.float32).astype(np.float64)
    assert wire.tensor_to_json(f) == ref.tensor_to_json(f)


def test_tensor_json_reads_bit_identical(ref):
    a = np.concatenate([npo.fill_random([500], 9), np.array(SPECIAL)]).reshape(-1, 1)
    text = ref.tensor_to_json(a)
    b = wire.tensor_from_json(text)
    assert b.shape == a.shape and np.array_equal(b.view(np.int64), a.view(np.int64))
    # whitespace / key order the reference's nlohmann reader also accepts
    j = json.loads(text)
    loose = json.dumps({"shape": j["shape"], "data": j["data"]}, indent=2)
    assert np.array_equal(wire.tensor_from_json(loose), ref.tensor_from_json(loose))


def test_tensor_json_errors(ref):
    with pytest.raises(ce.ShapeError):
        wire.tensor_from_json('{"shape":[2,2],"data":[1,2,3]}')  # tensor.cpp:143-144
    with pytest.raises(ce.ParseError):
        wire.tensor_from_json('{"shape":[2,2],"data":[1,2,3,4]')
    with pytest.raises(ce.ParseError):
        wire.tensor_from_json('{"data":[1]}')


def test_tensor_binary_matches_reference(ref):
    for shape, seed in [([3, 4], 1), ([2, 3, 5], 7), ([7], 2)]:
        a = npo.fill_random(shape, seed)
        raw = wire.tensor_to_binary(a)
        assert raw == ref.tensor_to_binary(a)
        b = wire.tensor_from_binary(raw)
        assert np.array_equal(b, a) and b.shape == a.shape
    with pytest.raises(ce.ShapeError):
        wire.tensor_from_binary(wire.tensor_to_binary(np.ones((2, 3)))[:-8])  # truncated stream


LAYERS = [
    '{"kind":"CP","T":[64],"S":[64],"H":3,"W":3,"Hp":32,"Wp":32,"B":8,"rank":16}',
    '{"kind":"TK","T":256,"S":256,"H":3,"W":3,"Hp":14,"Wp":14,"B":128,"rank":[57,57]}',
    '{"kind":"TT","T":[256],"S":[256],"H":3,"W":3,"Hp":14,"Wp":14,"rank":65}',
    '{"kind":"RTR","T":[4,4,8],"S":[4,4,4],"H":3,"W":3,"Hp":28,"Wp":28,"B":256,"rank":10}',
    '{"kind":"standard","T":[16],"S":[8],"H":3,"W":3,"Hp":8,"Wp":8,"B":2}',
    '{"kind":"HT","T":[2,2,2],"S":[2,2,2],"H":3,"W":3,"Hp":8,"Wp":8,"B":1,"rank":3}',
]


@pytest.mark.parametrize("text", LAYERS)
def test_layer_json_round_trip_matches_reference(ref, text):
    ours = wire.layer_to_json(wire.layer_from_json(text))
    assert ours == ref.layer_json_roundtrip(text)


def test_layer_json_errors(ref):
    for bad in ['{"kind":"nope","T":[4],"S":[4],"H":3,"W":3,"Hp":8,"Wp":8}',
                '{"kind":"CP","T":[4],"S":[4],"H":3,"W":3,"Hp":8}',
                '{"kind":"CP","T":[4],"S":[4],"H":3,"W":3,"Hp":8,"Wp":8,"rank":[1,2]}']:
        with pytest.raises(Exception):
            ref.layer_json_roundtrip(bad)
        with pytest.raises(ce.CeError):
            wire.layer_from_json(bad)


def test_number_formatting_random_bit_patterns(ref):
    """Grisu2 digit generation (nlohmann's dump, which the reference uses) over random
    finite doubles of every exponent, subnormals included: byte-identical."""
    rng = np.random.default_rng(1234)
    bits = rng.integers(0, 2 ** 63 - 1, size=20000, dtype=np.int64)
    vals = bits.view(np.float64)
    vals = vals[np.isfinite(vals)]
    sub = (rng.integers(1, 2 ** 52, size=500, dtype=np.int64)).view(np.float64)
    a = np.concatenate([vals, -vals[:1000], sub])
    assert wire.tensor_to_json(a) == ref.tensor_to_json(a)
