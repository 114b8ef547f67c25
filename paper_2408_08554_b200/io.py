"""On-disk weight formats of the reference -> device-resident engine weights
(the offline weight pipeline).

Formats (all little-endian), as written by the reference:
  ABQT  QuantizedTensor      include/abq/io.hpp:64-100  (write_quantized / read_quantized)
        "ABQT" u16 version=1, u8 bits, u8 scheme, u8 granularity, u32 rows, u32 cols,
        f32 scales[groups], i32 zero_points[groups], u8 codes[rows*cols];
        groups = 1 (per-tensor) or rows
  ABQP  BitPlaneMatrix       include/abq/io.hpp:102-124 (write_planes / read_planes)
        "ABQP" u16 version=1, u8 planes, u32 rows, u32 cols, u32 words_per_row,
        u64 words[planes*rows*words_per_row]
  ABQZ  offline model bundle tools/abqtool.cpp:211-237  (write_bundle)
        "ABQZ" u16 version=1, u32 count, then per layer: u16 name_len, name,
        an ABQT blob, an ABQP blob (bitpack of the same codes)

Parsing is host-side numpy (it runs without a GPU); `load_weights` /
`load_bundle` turn the records into `PackedWeights` resident in HBM -- the
ABQP planes uploaded as-is (or bit-packed on the device from ABQT codes),
colsum_b recovered on the device from the planes, and the decode / prefill
layouts prepacked once.  Errors follow io.hpp: `IoError` with the reference's
messages ("bad magic, expected ABQT", "ABQT: unsupported version", "unexpected
end of file", "ABQT: truncated code block", "ABQP: inconsistent words_per_row")
and the `ValueError`s of QuantizedTensor::validate (quantizer.hpp:98-106).
"""
from __future__ import annotations

import dataclasses
import io as _pyio
import struct
from typing import BinaryIO, Dict, List, Optional, Tuple, Union

import numpy as np

from .api import ASYMMETRIC, PER_TENSOR, IoError, QuantSpec, ValueError  # noqa: A004

FORMAT_VERSION = 1


@dataclasses.dataclass
class HostQuantized:
    """An ABQT record on the host: QuantizedTensor (quantizer.hpp:81-107) with
    its codes in a numpy array; scales are the file's f32 values as float64."""
    codes: np.ndarray        # uint8 [rows, cols]
    scales: np.ndarray       # float64 [groups]
    zero_points: np.ndarray  # int32 [groups]
    spec: QuantSpec

    def rows(self) -> int:
        return self.codes.shape[0]

    def cols(self) -> int:
        return self.codes.shape[1]

    def validate(self) -> None:
        """QuantizedTensor::validate (quantizer.hpp:98-106)."""
        self.spec.validate()
        max_code = self.spec.levels() - 1
        bad = np.flatnonzero(self.codes.reshape(-1) > max_code)
        if bad.size:
            raise ValueError(f"QuantizedTensor: code out of range at flat index {int(bad[0])}")
        want = 1 if self.spec.granularity == PER_TENSOR else self.rows()
        if self.scales.size != want or self.zero_points.size != want:
            raise ValueError("QuantizedTensor: scale/zero_point count does not match granularity")


@dataclasses.dataclass
class HostPlanes:
    """An ABQP record on the host: BitPlaneMatrix (bitplane.hpp:15-44)."""
    planes: int
    rows: int
    cols: int
    words: np.ndarray  # uint64 [planes, rows, words_per_row]

    @property
    def words_per_row(self) -> int:
        return (self.cols + 63) // 64


def _read(f: BinaryIO, n: int) -> bytes:
    b = f.read(n)
    if len(b) != n:
        raise IoError("unexpected end of file")
    return b


def _get(f: BinaryIO, fmt: str):
    return struct.unpack("<" + fmt, _read(f, struct.calcsize("<" + fmt)))[0]


def _expect_magic(f: BinaryIO, magic: bytes) -> None:
    b = f.read(4)
    if b != magic:
        raise IoError("bad magic, expected " + magic.decode())


def read_quantized(f: BinaryIO) -> HostQuantized:
    """read_quantized  io.hpp:78-100."""
    _expect_magic(f, b"ABQT")
    if _get(f, "H") != FORMAT_VERSION:
        raise IoError("ABQT: unsupported version")
    bits, scheme, gran = _get(f, "B"), _get(f, "B"), _get(f, "B")
    rows, cols = _get(f, "I"), _get(f, "I")
    groups = 1 if gran == PER_TENSOR else rows
    scales = np.frombuffer(_read(f, 4 * groups), dtype="<f4").astype(np.float64)
    zps = np.frombuffer(_read(f, 4 * groups), dtype="<i4").astype(np.int32)
    raw = f.read(rows * cols)
    if len(raw) != rows * cols:
        raise IoError("ABQT: truncated code block")
    q = HostQuantized(np.frombuffer(raw, dtype=np.uint8).reshape(rows, cols).copy(), scales, zps,
                      QuantSpec(bits=bits, scheme=scheme, granularity=gran))
    q.validate()
    return q


def write_quantized(f: BinaryIO, q: HostQuantized) -> None:
    """write_quantized  io.hpp:64-76 (scales stored as f32, like the reference)."""
    f.write(b"ABQT")
    f.write(struct.pack("<HBBBII", FORMAT_VERSION, q.spec.bits, q.spec.scheme, q.spec.granularity,
                        q.rows(), q.cols()))
    f.write(np.asarray(q.scales, dtype="<f4").tobytes())
    f.write(np.asarray(q.zero_points, dtype="<i4").tobytes())
    f.write(np.ascontiguousarray(q.codes, dtype=np.uint8).tobytes())


def read_planes(f: BinaryIO) -> HostPlanes:
    """read_planes  io.hpp:112-124."""
    _expect_magic(f, b"ABQP")
    if _get(f, "H") != FORMAT_VERSION:
        raise IoError("ABQP: unsupported version")
    planes, rows, cols, wpr = _get(f, "B"), _get(f, "I"), _get(f, "I"), _get(f, "I")
    if wpr != (cols + 63) // 64:
        raise IoError("ABQP: inconsistent words_per_row")
    n = planes * rows * wpr
    words = np.frombuffer(_read(f, 8 * n), dtype="<u8").reshape(planes, rows, wpr).copy()
    return HostPlanes(planes, rows, cols, words)


def write_planes(f: BinaryIO, p: HostPlanes) -> None:
    """write_planes  io.hpp:102-110."""
    f.write(b"ABQP")
    f.write(struct.pack("<HBIII", FORMAT_VERSION, p.planes, p.rows, p.cols, p.words_per_row))
    f.write(np.ascontiguousarray(p.words, dtype="<u8").tobytes())


def read_bundle(f: Union[str, BinaryIO]) -> List[Tuple[str, HostQuantized, HostPlanes]]:
    """ABQZ bundle (abqtool.cpp:211-237): [(name, ABQT record, ABQP record)]."""
    if isinstance(f, str):
        with open(f, "rb") as fh:
            return read_bundle(_pyio.BytesIO(fh.read()))
    _expect_magic(f, b"ABQZ")
    if _get(f, "H") != FORMAT_VERSION:
        raise IoError("ABQZ: unsupported version")
    out = []
    for _ in range(_get(f, "I")):
        name = _read(f, _get(f, "H")).decode()
        q = read_quantized(f)
        p = read_planes(f)
        if (p.rows, p.cols, p.planes) != (q.rows(), q.cols(), q.spec.planes()):
            raise IoError(f"ABQZ: layer {name}: planes do not match the quantized tensor")
        out.append((name, q, p))
    return out


def write_bundle(f: BinaryIO, layers: List[Tuple[str, HostQuantized, HostPlanes]]) -> None:
    f.write(b"ABQZ")
    f.write(struct.pack("<HI", FORMAT_VERSION, len(layers)))
    for name, q, p in layers:
        nb = name.encode()
        f.write(struct.pack("<H", len(nb)) + nb)
        write_quantized(f, q)
        write_planes(f, p)


def host_bitpack(codes: np.ndarray, planes: int) -> HostPlanes:
    """bitpack (bitplane.hpp:47-64) on the host, for files written from codes
    (test / tooling helper; the engine packs on the device)."""
    rows, cols = codes.shape
    wpr = (cols + 63) // 64
    padded = np.zeros((rows, wpr * 64), dtype=np.uint8)
    padded[:, :cols] = codes
    out = np.zeros((planes, rows, wpr), dtype=np.uint64)
    for s in range(planes):
        bits = ((padded >> s) & 1).astype(np.uint64).reshape(rows, wpr, 64)
        out[s] = (bits << np.arange(64, dtype=np.uint64)).sum(axis=2, dtype=np.uint64)
    return HostPlanes(planes, rows, cols, out)


def load_weights(q: HostQuantized, p: Optional[HostPlanes] = None, frag: bool = True, tc: bool = True):
    """One layer's records -> device-resident PackedWeights: the ABQP planes
    uploaded as-is when given (else packed on the device from the codes),
    colsum_b recovered on the device from the planes, decode (frag) and
    prefill (tc) layouts prepacked once."""
    from . import api
    if p is None:
        pm = api.bitpack(q.codes, q.spec.planes())
    else:
        pm = api.BitPlaneMatrix.from_numpy(p.words, p.cols)
    return api.PackedWeights.from_planes(pm, q.scales, q.zero_points, per_tensor=q.spec.granularity == PER_TENSOR,
                                         frag=frag, tc=tc)


def load_bundle(path: str, frag: bool = True, tc: bool = True) -> Dict[str, object]:
    """ABQZ bundle -> {layer name: PackedWeights} resident in HBM."""
    return {name: load_weights(q, p, frag, tc) for name, q, p in read_bundle(path)}


__all__ = ["HostQuantized", "HostPlanes", "read_quantized", "write_quantized", "read_planes", "write_planes",
           "read_bundle", "write_bundle", "host_bitpack", "load_weights", "load_bundle", "ASYMMETRIC"]
