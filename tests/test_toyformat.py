"""toy-json / toy-binary codec parity with the reference (golden encodings
produced by pkg/src/modelci/converter/toyformat.py) and its corruption cases
(pkg/tests/test_toyformat.py)."""
import json
import zlib
from pathlib import Path

import pytest

from paper_2006_05096_b200 import toyformat
from paper_2006_05096_b200.errors import ToyFormatError

GOLD = json.loads((Path(__file__).parent / "golden" / "toy_codec.json").read_text())


def test_binary_encoding_bit_identical_to_reference():
    for case in GOLD:
        assert toyformat.encode_binary(case["graph"]).hex() == case["binary_hex"]


def test_canonical_json_identical_to_reference():
    for case in GOLD:
        assert toyformat.canonical_json(case["graph"]).decode() == case["canonical"]


def test_decode_reference_bytes_round_trip():
    for case in GOLD:
        g = toyformat.decode_binary(bytes.fromhex(case["binary_hex"]))
        assert toyformat.canonical_json(g).decode() == case["canonical"]


def test_tricky_weights_exact():
    tricky = [0.1, 1e-300, -1e300, 2**53 + 1.0, 3.141592653589793]
    g = {"layers": [{"op": "linear", "in_dim": 1, "out_dim": 5, "weights": tricky}]}
    assert toyformat.decode_binary(toyformat.encode_binary(g))["layers"][0]["weights"] == tricky


def test_corruption():
    g = {"layers": [{"op": "linear", "in_dim": 2, "out_dim": 2, "weights": [0.5] * 4}]}
    data = bytearray(toyformat.encode_binary(g))
    data[10] ^= 0xFF
    with pytest.raises(ToyFormatError, match="CRC"):
        toyformat.decode_binary(bytes(data))
    with pytest.raises(ToyFormatError, match="magic"):
        toyformat.decode_binary(b"NOPE" + b"\0" * 16)
    with pytest.raises(ToyFormatError):
        toyformat.decode_binary(toyformat.encode_binary(g)[:8])
    payload = toyformat.encode_binary(g)[4:-4] + b"\x99"
    with pytest.raises(ToyFormatError):
        toyformat.decode_binary(toyformat.MAGIC + payload + zlib.crc32(payload).to_bytes(4, "little"))
    with pytest.raises(ToyFormatError):
        toyformat.parse_json(b"{not json")


@pytest.mark.parametrize("graph", [
    {}, {"layers": []},
    {"layers": [{"op": "", "in_dim": 1, "out_dim": 1, "weights": []}]},
    {"layers": [{"op": "x", "in_dim": 0, "out_dim": 1, "weights": []}]},
    {"layers": [{"op": "x", "in_dim": 1, "out_dim": 1, "weights": [float("nan")]}]},
    {"layers": [{"op": "x", "in_dim": 1, "out_dim": 1, "weights": [], "bogus": 1}]},
])
def test_invalid_graphs(graph):
    with pytest.raises(ToyFormatError):
        toyformat.validate_graph(graph)


def test_load_model_sniffs_and_dims():
    g = {"layers": [{"op": "linear", "in_dim": 3, "out_dim": 5, "weights": []},
                    {"op": "linear", "in_dim": 5, "out_dim": 2, "weights": []}]}
    assert toyformat.model_dims(toyformat.load_model(toyformat.encode_binary(g))) == (3, 2)
    assert toyformat.model_dims(toyformat.load_model(toyformat.canonical_json(g))) == (3, 2)
