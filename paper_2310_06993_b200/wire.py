"""Datagram framing for a lossy inter-node path, on the GPU.

The reference frames every shard into datagrams of at most ``MAX_PAYLOAD``
gradient bytes behind a 9-byte big-endian header
(``/root/reference/pkg/src/ubar/wire.py:36-85,176-208``).  On one NVSwitch
box the shards move through peer memory and no header is needed; for a
datagram transport between boxes (§8(f) rank 4) the framing runs here as
kernels (``optr_packetize`` / ``optr_depacketize``) straight from / into the
device shard, with the host-side header codec kept for callers that parse
single packets.

Packet layout in device memory: packet ``k`` occupies ``stride`` bytes at
``k * stride``: the header, then ``min(max_payload, bytes left)`` payload
bytes (the shard's float32 values, little-endian as numpy's ``tobytes``).
"""

from __future__ import annotations

from dataclasses import dataclass

from ._lib import check, lib

HEADER_LEN = 9
MAX_PAYLOAD = 1400
ENTRY_BYTES = 4

__all__ = ["HEADER_LEN", "MAX_PAYLOAD", "ENTRY_BYTES", "HeaderError", "PacketHeader", "encode_header",
           "decode_header", "quantize_timeout", "dequantize_timeout", "packets_for_bytes", "packetize",
           "depacketize"]


class HeaderError(ValueError):
    """Out-of-range header field or truncated header (wire.py:28-29)."""


@dataclass(frozen=True)
class PacketHeader:
    """wire.py:36-53; ``incast`` 0 means unchanged."""

    bucket_id: int
    byte_offset: int
    timeout_share: int = 0
    last_percentile: bool = False
    incast: int = 0

    def __post_init__(self):
        for name, value, hi in (("bucket_id", self.bucket_id, 0xFFFF), ("byte_offset", self.byte_offset, 0xFFFFFFFF),
                                ("timeout_share", self.timeout_share, 0xFF), ("incast", self.incast, 127)):
            if not 0 <= value <= hi:
                raise HeaderError(f"{name} out of range: {value}")


def encode_header(h: PacketHeader) -> bytes:
    """9 bytes: u16 bucket, u32 offset, u8 timeout, u8 flags, u8 reserved (BE)."""
    flags = int(bool(h.last_percentile)) | (h.incast << 1)
    return (h.bucket_id.to_bytes(2, "big") + h.byte_offset.to_bytes(4, "big")
            + bytes((h.timeout_share, flags, 0)))


def decode_header(b: bytes) -> PacketHeader:
    if len(b) < HEADER_LEN:
        raise HeaderError(f"need {HEADER_LEN} header bytes, got {len(b)}")
    if b[8] != 0:
        raise HeaderError(f"reserved header byte must be zero, got {b[8]}")
    return PacketHeader(bucket_id=int.from_bytes(b[0:2], "big"), byte_offset=int.from_bytes(b[2:6], "big"),
                        timeout_share=b[6], last_percentile=bool(b[7] & 1), incast=b[7] >> 1)


def quantize_timeout(t: float, t_b: float) -> int:
    """A duration in 1/255 units of the hard bound (wire.py:76-80)."""
    return 0 if t_b <= 0 else min(255, max(0, round(255.0 * t / t_b)))


def dequantize_timeout(share: int, t_b: float) -> float:
    return (share / 255.0) * t_b


def packets_for_bytes(n_bytes: int, max_payload: int = MAX_PAYLOAD) -> int:
    return 0 if n_bytes <= 0 else -(-n_bytes // max_payload)


def _stream(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def packetize(shard, bucket_id: int, base_offset: int = 0, max_payload: int = MAX_PAYLOAD,
              timeout_share: int = 0, incast: int = 0):
    """Frame a CUDA float32 shard into ``[n_packets, HEADER_LEN + max_payload]``
    uint8 packets (wire.py:183-208 iter_packets + encode_header); the last
    packet's unused tail bytes are zero."""
    import torch

    shard = shard.to(torch.float32).contiguous()
    total = packets_for_bytes(shard.numel() * ENTRY_BYTES, max_payload)
    stride = HEADER_LEN + max_payload
    out = torch.zeros((total, stride), dtype=torch.uint8, device=shard.device)
    check(lib().optr_packetize(shard.data_ptr() if shard.numel() else None, shard.numel(), int(bucket_id),
                               int(base_offset), int(max_payload), int(timeout_share), int(incast),
                               out.data_ptr() if total else None, stride, _stream(shard)), "packetize")
    return out


def depacketize(packets, n_entries: int, bucket_id: int, base_offset: int = 0, max_payload: int = MAX_PAYLOAD,
                delivered=None):
    """Reassemble a shard from received packets (rows of ``packets``; a False
    in ``delivered`` = dropped): zero-filled entries plus received flags, as
    the reference's receive buffers (simdriver.py:245-247,258-272).  Returns
    ``(entries, received, bad_headers)``."""
    import torch

    dev = packets.device
    entries = torch.empty(n_entries, dtype=torch.float32, device=dev)
    mask = torch.empty(n_entries, dtype=torch.uint8, device=dev)
    errors = torch.zeros(1, dtype=torch.int32, device=dev)
    d = None
    if delivered is not None:
        d = torch.as_tensor(delivered, dtype=torch.uint8, device=dev).contiguous()
    packets = packets.contiguous()
    check(lib().optr_depacketize(packets.data_ptr() if packets.numel() else None, packets.shape[0],
                                 packets.shape[1] if packets.dim() == 2 else HEADER_LEN + max_payload,
                                 d.data_ptr() if d is not None else None, int(bucket_id), int(base_offset),
                                 int(max_payload), entries.data_ptr() if n_entries else None,
                                 mask.data_ptr() if n_entries else None, n_entries, errors.data_ptr(),
                                 _stream(packets)), "depacketize")
    return entries, mask.bool(), int(errors.item())
