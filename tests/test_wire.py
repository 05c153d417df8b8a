"""Datagram framing (paper_2310_06993_b200.wire) against the reference's own
packet bytes (tests/golden/wire.npz from wire.iter_packets + encode_header,
wire.py:36-85,183-208).  Host header codec on CPU; the GPU packetizer /
depacketizer byte-exact on the GPU."""

import numpy as np
import pytest

from golden_util import load
from paper_2310_06993_b200 import wire as W


def _packets(z, i):
    lens = z[f"lens_{i}"]
    raw = z[f"bytes_{i}"].tobytes()
    out, pos = [], 0
    for ln in lens:
        out.append(raw[pos:pos + int(ln)])
        pos += int(ln)
    return out


def test_header_codec_matches_reference_bytes():
    z = load("wire.npz")
    for i, (ne, bid, base, mp, ts, inc) in enumerate(z["cases"]):
        pk = _packets(z, i)
        total = W.packets_for_bytes(int(ne) * 4, int(mp))
        assert len(pk) == total
        for k, p in enumerate(pk):
            h = W.decode_header(p)
            assert (h.bucket_id, h.byte_offset, h.timeout_share, h.incast) == (bid, base + k * mp, ts, inc)
            assert h.last_percentile == (k >= total - max(1, total // 100))
            assert W.encode_header(h) == p[:W.HEADER_LEN]


def test_header_errors():
    with pytest.raises(W.HeaderError):
        W.PacketHeader(bucket_id=1 << 16, byte_offset=0)
    with pytest.raises(W.HeaderError):
        W.PacketHeader(bucket_id=0, byte_offset=0, incast=128)
    with pytest.raises(W.HeaderError):
        W.decode_header(b"\x00" * 8)
    with pytest.raises(W.HeaderError):
        W.decode_header(b"\x00" * 8 + b"\x01")
    assert W.quantize_timeout(0.5, 1.0) == 128 and W.quantize_timeout(2.0, 1.0) == 255
    assert W.quantize_timeout(1.0, 0.0) == 0


@pytest.mark.gpu
def test_gpu_packetizer_byte_exact_and_reassembly():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    z = load("wire.npz")
    for i, (ne, bid, base, mp, ts, inc) in enumerate(z["cases"]):
        x = torch.from_numpy(z[f"x_{i}"]).cuda()
        got = W.packetize(x, int(bid), int(base), int(mp), int(ts), int(inc)).cpu().numpy()
        want = _packets(z, i)
        assert got.shape[0] == len(want)
        for k, p in enumerate(want):
            np.testing.assert_array_equal(got[k, :len(p)], np.frombuffer(p, dtype=np.uint8))
        # drop every 7th packet: zero-filled entries, received flags cleared
        keep = np.ones(len(want), dtype=bool)
        keep[::7] = False
        ent, rcv, bad = W.depacketize(torch.from_numpy(got).cuda(), int(ne), int(bid), int(base), int(mp), keep)
        assert bad == 0
        epp = int(mp) // 4
        m = np.repeat(keep, epp)[: int(ne)]
        np.testing.assert_array_equal(rcv.cpu().numpy(), m)
        np.testing.assert_array_equal(ent.cpu().numpy(), np.where(m, z[f"x_{i}"], np.float32(0)))
        if len(want):  # a corrupted reserved byte / foreign bucket is rejected and counted
            bad_pk = torch.from_numpy(got.copy()).cuda()
            bad_pk[0, 8] = 1
            _e, r2, nbad = W.depacketize(bad_pk, int(ne), int(bid), int(base), int(mp))
            assert nbad == 1 and not r2[:min(epp, int(ne))].any()
            _e, _r, nbad = W.depacketize(torch.from_numpy(got).cuda(), int(ne), (int(bid) + 1) & 0xFFFF,
                                         int(base), int(mp))
            assert nbad == len(want)
