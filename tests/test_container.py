"""rs-tensor-container v1: byte-compatibility with files
written by the reference's own ``write_rs`` / ``write_reference``
(tests/golden/make_golden_next.py)."""
import hashlib
import os

import numpy as np
import pytest

from paper_1606_09218_b200 import container

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FILES = ["next_tiny_reference.rsc", "next_tiny_tucker.rsc", "next_C1_canonical.rsc"]


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", FILES)
def test_sections_round_trip_bit_exact(name):
    blob = _bytes(name)
    sec = container.decode_sections(blob, name)
    assert container.encode_sections(list(sec.items())) == blob


def test_reference_round_trip_bit_exact(tmp_path):
    ref = container.read_reference(os.path.join(GOLD, "next_tiny_reference.rsc"))
    assert ref.grid.n == 64 and ref.doubled is not None
    out = tmp_path / "ref.rsc"
    container.write_reference(ref, out)
    assert out.read_bytes() == _bytes("next_tiny_reference.rsc")


def test_canonical_rs_round_trip_bit_exact(tmp_path):
    rs = container.read_rs(os.path.join(GOLD, "next_C1_canonical.rsc"))
    assert rs.long.rank == 64 and rs.grid.n == 128
    out = tmp_path / "rs.rsc"
    container.write_rs(rs, out)
    assert out.read_bytes() == _bytes("next_C1_canonical.rsc")


def test_bad_containers_raise(tmp_path):
    from paper_1606_09218_b200.errors import ParseError
    with pytest.raises(ParseError):
        container.decode_sections(b"not a container")
    blob = _bytes("next_tiny_tucker.rsc")
    with pytest.raises(ParseError):
        container.decode_sections(blob[:-5])
    p = tmp_path / "x.rsc"
    p.write_bytes(_bytes("next_tiny_reference.rsc"))
    with pytest.raises(ParseError):
        container.read_rs(p)


@pytest.mark.gpu
def test_tucker_rs_round_trip_bit_exact(cuda, tmp_path):
    rs = container.read_rs(os.path.join(GOLD, "next_tiny_tucker.rsc"))
    out = tmp_path / "rs.rsc"
    container.write_rs(rs, out)
    assert out.read_bytes() == _bytes("next_tiny_tucker.rsc")


@pytest.mark.gpu
def test_container_of_a_device_build(cuda, tmp_path):
    """A GPU-built RS tensor written and read back assembles the same grid."""
    import paper_1606_09218_b200 as rt
    from oracle import rs_oracle as orc
    c = orc.small_case(n=32, count=24, seed=5)
    box = rt.Box3(c["b"])
    cfg = rt.AssemblyConfig(grid=rt.Grid3(32, box), kernel=rt.RadialKernel("newton", 1.0), M=15,
                            split_index=7, sigma=1.0, delta=1e-6, long_format="tucker",
                            reduction=rt.ReductionConfig(eps=1e-8, max_sweeps=0), max_overlap=None)
    res = rt.build_rs(rt.ParticleSystem(c["positions"], c["charges"], box), cfg)
    p = tmp_path / "built.rsc"
    container.write_rs(res.rs, p)
    back = container.read_rs(p)
    g0 = rt.dense_rs(res.rs, limit=1 << 30)
    g1 = rt.dense_rs(back, limit=1 << 30)
    assert np.array_equal(g0, g1)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == hashlib.sha256(
        container.encode_sections(container.rs_sections(back))).hexdigest()


@pytest.mark.gpu
def test_grad_long_matches_reference(cuda):
    """grad_long of the reference's RS tensors, read from
    the reference-written containers: dense components vs the reference."""
    import paper_1606_09218_b200 as rt
    rs = container.read_rs(os.path.join(GOLD, "next_tiny_tucker.rsc"))
    g = np.load(os.path.join(GOLD, "next_tiny_grad.npz"))
    for a, c in enumerate(rt.grad_long(rs)):
        ref = g[f"g{a}"]
        assert np.max(np.abs(c.dense(limit=1 << 20) - ref)) <= 1e-12 * np.abs(ref).max()
    rs = container.read_rs(os.path.join(GOLD, "next_C1_canonical.rsc"))
    g = np.load(os.path.join(GOLD, "next_C1_canonical_grad.npz"))
    s = g["sample_idx"]
    for a, c in enumerate(rt.grad_long(rs)):
        d = c.dense(limit=1 << 24)[s[:, 0], s[:, 1], s[:, 2]]
        ref = g[f"g{a}"]
        assert np.max(np.abs(d - ref)) <= 1e-12 * np.abs(ref).max()
