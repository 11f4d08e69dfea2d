"""Handle images (sable_serialize / sable_deserialize):
compile once, run many.  A loaded handle must behave as
the inspected one: identical image bytes on re-serialisation, identical
partition export, bitwise identical y, the same info; corrupted or truncated
images fail with SABLE_E_FORMAT."""
import numpy as np
import pytest

import gen
import oracle
from parity import assert_y_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sable():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_00829_b200 import sable as s
    return s


def make(sable, s, rank=0, world=1, delta=None):
    inp = s.vbr_input("rect")
    arrays = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()
              if isinstance(v, np.ndarray)}
    return sable.VbrMatrix(arrays, s.nrows, s.ncols, delta=s.delta if delta is None else delta,
                           rank=rank, world=world)


@pytest.mark.parametrize("name,scale,rank,world", [("c1", 1.0, 0, 1), ("c2", 0.02, 0, 1),
                                                   ("c3", 0.01, 1, 3), ("c5", 1 / 512, 0, 1)])
def test_round_trip(sable, name, scale, rank, world):
    s = gen.make(name, scale=scale)
    A = make(sable, s, rank, world)
    img = A.serialize()
    B = sable.VbrMatrix.from_image(img)
    try:
        assert B.serialize() == img  # byte-identical round trip
        assert A.serialize() == img  # serialising does not change the handle
        ia, ib = dict(A.info), dict(B.info)
        assert ia == ib
        ea, eb = A.export(), B.export()
        for k in ea:
            np.testing.assert_array_equal(ea[k].view(np.uint8), eb[k].view(np.uint8), err_msg=k)
        x = torch.from_numpy(s.x).cuda()
        ya = A.spmv(x).cpu().numpy()
        yb = B.spmv(x).cpu().numpy()
        np.testing.assert_array_equal(ya.view(np.uint8), yb.view(np.uint8))
        # and it is still the product (the loaded handle is usable on its own)
        A.close()
        r0, r1 = ib["row_begin"], ib["row_end"]
        yo, so = oracle.spmv_rows(s.rowptr(), s.J, s.V.astype(np.float64),
                                  s.x.astype(np.float64), np.arange(r0, r1))
        yb2 = B.spmv(x).cpu().numpy()
        assert_y_close(yb2, yo, so, s.dtype, f"{name}/image")
        yh = B.spmv_host(s.x)
        np.testing.assert_array_equal(yh.view(np.uint8), yb.view(np.uint8))
    finally:
        A.close()
        B.close()


def test_image_errors(sable):
    s = gen.make("c1")
    A = make(sable, s)
    img = bytearray(A.serialize())
    A.close()
    bad = bytearray(img)
    bad[-3] ^= 0x40  # payload bit flip -> checksum
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(bad))
    assert e.value.status == sable.SABLE_E_FORMAT
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(img[:-8]))  # truncated
    assert e.value.status == sable.SABLE_E_FORMAT
    bad = bytearray(img)
    bad[0:8] = b"NOTSABLE"
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(bad))
    assert e.value.status == sable.SABLE_E_FORMAT
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(img[:16]))
    assert e.value.status == sable.SABLE_E_INVALID_ARG


def test_suitability_survives(sable):
    # delta = 101: nothing dense -> not suitable; the image keeps it
    s = gen.make("c1")
    A = make(sable, s, delta=101)
    B = sable.VbrMatrix.from_image(A.serialize())
    assert A.info["suitable"] == B.info["suitable"] == 0
    A.close()
    B.close()


def _fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_image_semantic_checks(sable):
    """An image whose checksum is right but whose content is not (a header
    field out of range, or a unit index past its arrays, with the payload
    checksum recomputed) is rejected with SABLE_E_FORMAT before any upload."""
    import struct
    s = gen.make("c1")
    A = make(sable, s)
    img = bytes(A.serialize())
    A.close()
    hdr = struct.unpack_from("<i", img, 12)[0]
    fnv_at = hdr - 8 * 22 - 8  # ImageHeader of serial.cu: ..., payload_fnv, section_bytes[22]
    # executor configuration: rem_rows (cfg at byte 96: pf, ustage, rem_rows, batch)
    bad = bytearray(img)
    struct.pack_into("<i", bad, 104, 99)
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(bad))
    assert e.value.status == sable.SABLE_E_FORMAT
    # unit 0 (section 0, right after the header): rows past the local rows
    bad = bytearray(img)
    struct.pack_into("<i", bad, hdr + 4, 1 << 30)  # row0
    struct.pack_into("<Q", bad, fnv_at, _fnv1a(bytes(bad[hdr:])))
    with pytest.raises(sable.SableError) as e:
        sable.VbrMatrix.from_image(bytes(bad))
    assert e.value.status == sable.SABLE_E_FORMAT
    assert "unit 0" in str(e.value)
