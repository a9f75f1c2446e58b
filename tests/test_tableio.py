"""ARVT table files: files written by the reference's own export_table
(tests/golden/arvt, made by make_golden.py) load here, and our writer
reproduces them byte for byte (tableio.py:30-223)."""

import os

import numpy as np
import pytest

ARVT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "arvt")


@pytest.fixture(scope="module")
def tio():
    from paper_2012_09715_b200 import tableio

    return tio_mod(tableio)


def tio_mod(m):
    return m


def ours(name):
    import paper_2012_09715_b200 as arv

    return {
        "constant_q10": arv.load_table("constant_q10_l1"),
        "dyadic_linear_k15": arv.load_table("dyadic_linear_k15"),
        "dyadic_cubic_k15": arv.load_table("dyadic_cubic_k15"),
        "ncchi2_cir_k16": arv.load_table("ncchi2_cir_k16_stacks"),
    }[name]


def payload(t):
    for attr in ("values", "coeffs", "eval_stacks"):
        if hasattr(t, attr):
            return np.asarray(getattr(t, attr))
    raise AssertionError(type(t))


NAMES = ["constant_q10", "dyadic_linear_k15", "dyadic_cubic_k15", "ncchi2_cir_k16"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("ext", [".arvt", ".txt"])
def test_reads_reference_files(tio, name, ext):
    t = tio.import_table(os.path.join(ARVT, name + ext))
    ref = ours(name)
    assert type(t).__name__ == type(ref).__name__
    assert np.array_equal(payload(t), payload(ref))
    if hasattr(ref, "nu"):
        assert t.nu == ref.nu


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("fmt,ext", [("binary", ".arvt"), ("text", ".txt")])
def test_writes_reference_bytes(tio, tmp_path, name, fmt, ext):
    p = tmp_path / ("x" + ext)
    tio.export_table(ours(name), p, format=fmt)
    with open(os.path.join(ARVT, name + ext), "rb") as fh:
        assert p.read_bytes() == fh.read()


def test_subdyadic_round_trip(tio, tmp_path):
    import paper_2012_09715_b200 as arv

    t = arv.load_table("subdyadic_linear_k16_s8")
    for fmt in ("binary", "text"):
        p = tmp_path / f"s.{fmt}"
        tio.export_table(t, p, format=fmt)
        back = tio.import_table(p)
        assert isinstance(back, arv.SubDyadicTable) and back.sub_bits == 3
        assert np.array_equal(back.coeffs, t.coeffs)


def test_errors(tio, tmp_path):
    import paper_2012_09715_b200 as arv

    good = open(os.path.join(ARVT, "dyadic_linear_k15.arvt"), "rb").read()
    cases = {
        "magic": (b"XXXX" + good[4:], arv.BadMagicError),
        "version": (good[:4] + b"\x02\x00" + good[6:], arv.VersionError),
        "crc": (good[:20] + bytes([good[20] ^ 1]) + good[21:], arv.ChecksumError),
        "short": (good[:10], arv.TableIOError),
    }
    for key, (blob, exc) in cases.items():
        p = tmp_path / key
        p.write_bytes(blob)
        with pytest.raises(exc):
            tio.import_table(p)
    with pytest.raises(arv.ConfigError):
        tio.export_table(object(), tmp_path / "o")
