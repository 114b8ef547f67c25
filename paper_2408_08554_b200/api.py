"""Python mirror of the reference operator API for the hot path.

Same names, argument meaning and error behaviour as the reference's C++
functions in namespace ``abq`` (paths relative to /root/reference/proj):

  core.hpp:13-36        Error / ShapeError / ValueError / OverflowError / IoError
  quantizer.hpp:37-254  QuantSpec, QuantizedTensor, quantize, quantize_balanced, dequantize*
  bitplane.hpp:15-96    BitPlaneMatrix, bitpack, unpack, bmma
  gemm.hpp:19-307       TileConfig, default_tile, GemmStats, fits_int32, engine_threads,
                        gemm_arbitrary(_wide), gemm_naive, zero_point_correct,
                        code_rowsums, quantized_linear
  tune.hpp:17-192       padding_redundancy, enumerate_tile_candidates, BenchRecord,
                        AutotuneResult, autotune (+ autotune_linear: the engine's own
                        schedules -- GEMV variant, prefill GEMM classic / stream-K)

Every numeric result is computed by the sm_100a kernels behind the C-ABI
(include/abq_cuda.h); tensors live on the GPU (torch CUDA storage is used for
device memory and streams only).  (*) dequantize is the reference's inverse
map and runs as a plain elementwise torch op on the device.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional

import numpy as np
import torch

from . import _lib as L

# ---------------------------------------------------------------------------
# errors (core.hpp:13-36)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class ValueError(Error, ValueError):  # noqa: A001 - mirrors abq::ValueError
    pass


class OverflowError(Error, OverflowError):  # noqa: A001 - mirrors abq::OverflowError
    pass


class IoError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {L.ABQ_ERR_SHAPE: ShapeError, L.ABQ_ERR_VALUE: ValueError,
           L.ABQ_ERR_OVERFLOW: OverflowError, L.ABQ_ERR_IO: IoError, L.ABQ_ERR_CUDA: CudaError}


def _check(status: int) -> None:
    if status != L.ABQ_OK:
        msg = L.lib().abq_last_error().decode()
        raise _STATUS.get(status, Error)(msg)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("engine tensors must live on the GPU")
    return t.data_ptr()


def _out_ptr(t: torch.Tensor) -> int:
    """device tensor, or pinned host tensor (its UVA address: the engine
    writes it over PCIe)"""
    return t.data_ptr() if (t.device.type == "cpu" and t.is_pinned()) else _ptr(t)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise CudaError("abq: no CUDA device available; the engine has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dtype) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    return x.to(device=_dev(), dtype=dtype).contiguous()


# ---------------------------------------------------------------------------
# quantizer (quantizer.hpp)
# ---------------------------------------------------------------------------
ASYMMETRIC, SYMMETRIC, BALANCED = L.ABQ_ASYMMETRIC, L.ABQ_SYMMETRIC, L.ABQ_BALANCED
PER_TENSOR, PER_CHANNEL, PER_TOKEN = L.ABQ_PER_TENSOR, L.ABQ_PER_CHANNEL, L.ABQ_PER_TOKEN


@dataclasses.dataclass
class QuantSpec:
    """QuantSpec  quantizer.hpp:37-71."""
    bits: int = 8
    scheme: int = ASYMMETRIC
    granularity: int = PER_TENSOR
    alpha: float = 1.0
    beta: float = 1.0

    def passthrough(self) -> bool:
        return self.bits >= 16

    def levels(self) -> int:
        return (1 << self.bits) + 1 if self.scheme == BALANCED else (1 << self.bits)

    def planes(self) -> int:
        lv, p = self.levels(), 0
        while (1 << p) < lv:
            p += 1
        return p

    def validate(self) -> None:
        if self.bits < 1 or (self.bits > 8 and not self.passthrough()):
            raise ValueError("QuantSpec: bits must be in [1,8] (or >=16 for passthrough)")
        if self.scheme == BALANCED and self.bits > 7 and not self.passthrough():
            raise ValueError("QuantSpec: balanced codes reach 2^bits and must fit one byte, so bits <= 7")
        if not (0.0 < self.alpha <= 1.0):
            raise ValueError("QuantSpec: alpha must be in (0,1]")
        if not (0.0 < self.beta <= 1.0):
            raise ValueError("QuantSpec: beta must be in (0,1]")

    def c(self) -> L.QuantSpecC:
        return L.QuantSpecC(self.bits, self.scheme, self.granularity, self.alpha, self.beta)


@dataclasses.dataclass
class QuantizedTensor:
    """QuantizedTensor  quantizer.hpp:81-107 (device tensors)."""
    codes: torch.Tensor          # uint8 rows x cols
    scales: torch.Tensor         # float64, 1 or rows
    zero_points: torch.Tensor    # int32, 1 or rows
    spec: QuantSpec

    def rows(self) -> int:
        return self.codes.shape[0]

    def cols(self) -> int:
        return self.codes.shape[1]

    def axis_of(self, i: int, j: int = 0) -> int:
        return 0 if self.spec.granularity == PER_TENSOR else i


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float16:
        return L.ABQ_F16
    if t.dtype == torch.float64:
        return L.ABQ_F64
    if t.dtype == torch.float32:
        return L.ABQ_F32
    raise ValueError(f"quantize: unsupported dtype {t.dtype}")


def quantize(x, spec: QuantSpec, comp: Optional[tuple] = None) -> QuantizedTensor:
    """quantize  quantizer.hpp:146-213 on the GPU (bit-exact FP64)."""
    spec.validate()
    if spec.passthrough():
        raise ValueError("quantize: passthrough spec cannot be materialized")
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.dtype not in (torch.float16, torch.float32, torch.float64):
        x = x.to(torch.float64)
    x = x.to(_dev()).contiguous()
    rows, cols = x.shape
    ca = cb = None
    if comp is not None:
        a, b = comp
        ca, cb = _to_dev(a, torch.float64), _to_dev(b, torch.float64)
        if ca.numel() != rows or cb.numel() != cols:
            raise ShapeError("quantize: compensation pair does not match matrix shape")
    groups = 1 if spec.granularity == PER_TENSOR else rows
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=x.device)
    scales = torch.empty(groups, dtype=torch.float64, device=x.device)
    zps = torch.empty(groups, dtype=torch.int32, device=x.device)
    cs = spec.c()
    _check(L.lib().abq_quantize(_ptr(x), _dtype_code(x), rows, cols, C.byref(cs), _ptr(ca), _ptr(cb),
                                _ptr(codes), _ptr(scales), _ptr(zps), _stream()))
    return QuantizedTensor(codes, scales, zps, dataclasses.replace(spec))


def quantize_balanced(x, bits: int, granularity: int = PER_TENSOR) -> QuantizedTensor:
    """quantize_balanced  quantizer.hpp:217-224."""
    return quantize(x, QuantSpec(bits=bits, scheme=BALANCED, granularity=granularity))


def dequantize(q: QuantizedTensor) -> torch.Tensor:
    """dequantize  quantizer.hpp:243-254: (code - z) * step in FP64."""
    idx = 0 if q.spec.granularity == PER_TENSOR else slice(None)
    s = q.scales[idx].reshape(-1, 1) if idx != 0 else q.scales[0]
    z = q.zero_points[idx].reshape(-1, 1).double() if idx != 0 else q.zero_points[0].double()
    return (q.codes.double() - z) * s


# ---------------------------------------------------------------------------
# bit planes (bitplane.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class BitPlaneMatrix:
    """BitPlaneMatrix  bitplane.hpp:15-44: data is [planes][rows][words_per_row]
    u64 words (stored in an int64 CUDA tensor), LSB-first, tail bits zero."""
    planes: int
    rows: int
    cols: int
    data: torch.Tensor

    @property
    def words_per_row(self) -> int:
        return (self.cols + 63) // 64

    @staticmethod
    def from_numpy(words: np.ndarray, cols: int) -> "BitPlaneMatrix":
        p, r, _ = words.shape
        return BitPlaneMatrix(p, r, cols, _to_dev(words.view(np.int64), torch.int64))

    def numpy(self) -> np.ndarray:
        return self.data.cpu().numpy().view(np.uint64)

    def __eq__(self, o) -> bool:
        return (self.planes, self.rows, self.cols) == (o.planes, o.rows, o.cols) and bool(
            torch.equal(self.data, o.data))


def _empty_planes(bits: int, rows: int, cols: int) -> torch.Tensor:
    return torch.empty((bits, rows, (cols + 63) // 64), dtype=torch.int64, device=_dev())


def bitpack(codes, bits: int) -> BitPlaneMatrix:
    """bitpack  bitplane.hpp:47-64 ([M,K] codes -> [bits,M,K] planes)."""
    codes = _to_dev(codes, torch.uint8)
    rows, cols = codes.shape
    out = _empty_planes(max(1, min(bits, 8)), rows, cols)
    _check(L.lib().abq_bitpack(_ptr(codes), rows, cols, bits, _ptr(out), _stream()))
    return BitPlaneMatrix(bits, rows, cols, out)


def unpack(m: BitPlaneMatrix) -> torch.Tensor:
    """unpack  bitplane.hpp:66-76."""
    codes = torch.empty((m.rows, m.cols), dtype=torch.uint8, device=_dev())
    _check(L.lib().abq_unpack(_ptr(m.data), m.planes, m.rows, m.cols, _ptr(codes), _stream()))
    return codes


def bmma(a: BitPlaneMatrix, a_plane: int, bt: BitPlaneMatrix, b_plane: int) -> torch.Tensor:
    """bmma  bitplane.hpp:81-96 (single plane pair AND + popcount)."""
    if a.cols != bt.cols:
        raise ShapeError("bmma: shared K dimension differs")
    out = torch.empty((a.rows, bt.rows), dtype=torch.int32, device=_dev())
    _check(L.lib().abq_bmma(_ptr(a.data), a.planes, a.rows, a_plane, _ptr(bt.data), bt.planes,
                            bt.rows, b_plane, a.cols, _ptr(out), _stream()))
    return out


def gemm_btc(a: BitPlaneMatrix, bt: BitPlaneMatrix) -> torch.Tensor:
    """The plane GEMM of gemm_arbitrary (gemm.hpp:94-146) on the b1 tensor-core
    path (mma.sync m16n8k256 .b1 and.popc): the measured comparator of the
    tcgen05 recombination GEMM.  Returns int32 [M][N]."""
    out = torch.empty((a.rows, bt.rows), dtype=torch.int32, device=_dev())
    _check(L.lib().abq_gemm_btc(_ptr(a.data), a.planes, a.rows, a.cols, _ptr(bt.data), bt.planes, bt.rows,
                                bt.cols, _ptr(out), _stream()))
    return out


# ---------------------------------------------------------------------------
# engine (gemm.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class TileConfig:
    """TileConfig  gemm.hpp:19-48."""
    BM: int = 64
    BN: int = 64
    BK: int = 512
    WM: int = 64
    WN: int = 64
    WK: int = 128
    mma_m = 8
    mma_n = 8
    mma_k = 128

    def c(self) -> L.TileConfigC:
        return L.TileConfigC(self.BM, self.BN, self.BK, self.WM, self.WN, self.WK)

    def valid(self, p: int, q: int) -> bool:
        return bool(L.lib().abq_tile_valid(C.byref(self.c()), p, q))

    def require_valid(self, p: int, q: int) -> None:
        if not self.valid(p, q):
            raise ValueError(
                f"TileConfig invalid for p={p} q={q}: BM={self.BM} BN={self.BN} BK={self.BK} "
                f"WM={self.WM} WN={self.WN} WK={self.WK}")

    def describe(self) -> str:
        return f"BM{self.BM}_BN{self.BN}_BK{self.BK}_WM{self.WM}_WN{self.WN}"


def tile_engine_plan(tile: TileConfig) -> tuple:
    """(token_tile, schedule) the engine runs gemm_arbitrary with for this tile
    (abq_tile_engine_plan): schedule is "stream_k" or "classic"."""
    tt, sc = C.c_int(0), C.c_int(0)
    _check(L.lib().abq_tile_engine_plan(C.byref(tile.c()), C.byref(tt), C.byref(sc)))
    return tt.value, {1: "classic", 2: "stream_k"}.get(sc.value, "auto")


def default_tile(p: int, q: int) -> TileConfig:
    """default_tile  gemm.hpp:51-59."""
    t = L.lib().abq_default_tile(p, q)
    return TileConfig(t.BM, t.BN, t.BK, t.WM, t.WN, t.WK)


@dataclasses.dataclass
class GemmStats:
    """GemmStats  gemm.hpp:61-64 (accumulated across calls)."""
    block_tiles: int = 0
    plane_pair_products: int = 0


def fits_int32(p: int, q: int, k: int) -> bool:
    """fits_int32  gemm.hpp:73-77."""
    return bool(L.lib().abq_fits_int32(p, q, k))


_engine_threads = [0]


def engine_threads() -> list:
    """engine_threads  gemm.hpp:81-84.  Kept for API parity: a process-global
    knob whose value never changes results; the GPU engine ignores it."""
    return _engine_threads


def padding_redundancy(m: int, p: int, mma_m: int) -> float:
    """padding_redundancy  tune.hpp:17-23."""
    out = C.c_double()
    _check(L.lib().abq_padding_redundancy(m, p, mma_m, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# tuning (tune.hpp)
# ---------------------------------------------------------------------------
_WARP_LAYOUTS = ((1, 1), (1, 2), (1, 4), (2, 2), (2, 4), (4, 4))  # tune.hpp:28-32


def _total_row_padding(m: int, p: int, bm: int, mma_m: int) -> int:
    """detail::total_row_padding  tune.hpp:35-44."""
    pad = 0
    for m0 in range(0, m, bm):
        e = p * min(bm, m - m0)
        pad += -(-e // mma_m) * mma_m - e
    return pad


def enumerate_tile_candidates(p: int, q: int, m: int, n: int, k: int) -> List[TileConfig]:
    """enumerate_tile_candidates  tune.hpp:51-92: warp layout x power-of-two inner
    tiles x BK grid, block tile derived from the layout, deduplicated, then only
    the block heights with the least row padding for (p, M).  Host logic; the
    validity check is the engine's (abq_tile_valid)."""
    if not (1 <= p <= 8 and 1 <= q <= 8):
        raise ValueError("enumerate_tile_candidates: p,q must be in [1,8]")
    seen, raw = set(), []
    for lm, ln in _WARP_LAYOUTS:
        for wm in (8, 16, 32, 64):
            for wn in (8, 16, 32, 64):
                for bk in (128, 256, 384, 512):
                    t = TileConfig(BM=-(-(lm * wm) // p), BN=-(-(ln * wn) // q), BK=bk, WM=wm, WN=wn,
                                   WK=TileConfig.mma_k)
                    if not t.valid(p, q):
                        continue
                    key = (t.BM, t.BN, t.BK, t.WM, t.WN)
                    if key in seen:
                        continue
                    seen.add(key)
                    raw.append(t)
    best = min((_total_row_padding(m, p, t.BM, TileConfig.mma_m) for t in raw), default=None)
    out = [t for t in raw if _total_row_padding(m, p, t.BM, TileConfig.mma_m) == best]
    return out or [default_tile(p, q)]


@dataclasses.dataclass
class BenchRecord:
    """BenchRecord  tune.hpp:94-105 (one CSV row per timed candidate)."""
    config_id: str = ""
    BM: int = 0
    BN: int = 0
    BK: int = 0
    WM: int = 0
    WN: int = 0
    p: int = 0
    q: int = 0
    M: int = 0
    N: int = 0
    K: int = 0
    median_us: float = 0.0
    tops: float = 0.0  # 2*M*N*K ops over the median latency

    @staticmethod
    def csv_header() -> str:
        return "config_id,BM,BN,BK,WM,WN,p,q,M,N,K,median_us,tops"

    def csv_row(self) -> str:
        return ",".join(str(v) for v in dataclasses.astuple(self))


@dataclasses.dataclass
class AutotuneResult:
    """AutotuneResult  tune.hpp:136-139 (best: a TileConfig for autotune, the
    schedule name for autotune_linear)."""
    best: object
    records: List[BenchRecord]


def tops_of(m: int, n: int, k: int, us: float) -> float:
    """detail::tops_of  tune.hpp:129-131."""
    return 2.0 * m * n * k / (us * 1e6)


def _time_median_us(fn, trials: int) -> float:
    """detail::time_median_us  tune.hpp:114-127 on the device: one discarded
    warm-up, then `trials` calls each bracketed by CUDA events on the current
    stream; median (mean of the middle two for even counts)."""
    fn()
    times = []
    st = torch.cuda.current_stream()
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    h = len(times) // 2
    return times[h] if len(times) % 2 else 0.5 * (times[h - 1] + times[h])


def _time_graph_us(fn, trials: int, reps: int = 20) -> float:
    """Per-call device time of `fn` replayed from a CUDA graph of `reps` calls
    (the serving path; eager timing would measure host launch overhead):
    median over `trials` replays bracketed by CUDA events."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3 / reps)
    times.sort()
    h = len(times) // 2
    return times[h] if len(times) % 2 else 0.5 * (times[h - 1] + times[h])


def autotune(candidates: List[TileConfig], a: "BitPlaneMatrix", bt: "BitPlaneMatrix",
             trials: int = 3) -> AutotuneResult:
    """autotune  tune.hpp:141-192: time every candidate through gemm_arbitrary
    (gemm_arbitrary_wide when the int32 bound does not hold), verify each result
    bit for bit against the first candidate's (a mismatch is a hard Error), and
    return the fastest.  Timing is device time (CUDA events) instead of the
    reference's steady_clock."""
    if not candidates:
        raise ValueError("autotune: no candidates")
    if trials < 3:
        raise ValueError("autotune: need at least 3 trials")
    wide = not fits_int32(a.planes, bt.planes, a.cols)
    fn = gemm_arbitrary_wide if wide else gemm_arbitrary
    reference, records, best = None, [], 0
    for ci, t in enumerate(candidates):
        t.require_valid(a.planes, bt.planes)
        got = [None]

        def run():
            got[0] = fn(a, bt, t)

        us = _time_median_us(run, trials)
        if ci == 0:
            reference = got[0]
        elif not torch.equal(got[0], reference):
            raise Error(f"autotune: config {t.describe()} disagrees with the reference result")
        rec = BenchRecord(t.describe(), t.BM, t.BN, t.BK, t.WM, t.WN, a.planes, bt.planes, a.rows, bt.rows,
                          a.cols, us, tops_of(a.rows, bt.rows, a.cols, us))
        if records and us < records[best].median_us:
            best = len(records)
        records.append(rec)
    return AutotuneResult(candidates[best], records)


GEMM_SCHEDULES = {"auto": 0, "classic": 1, "stream_k": 2}


def set_gemm_schedule(schedule: str) -> None:
    """Prefill GEMM schedule (abq_set_gemm_schedule): "auto", "classic" (one CTA
    per 128-channel row tile) or "stream_k" (all SMs share (row-tile, k-block)
    units).  Process-global; results do not depend on it."""
    if schedule not in GEMM_SCHEDULES:
        raise ValueError(f"set_gemm_schedule: unknown schedule {schedule!r}")
    _check(L.lib().abq_set_gemm_schedule(GEMM_SCHEDULES[schedule]))


def get_gemm_schedule() -> str:
    v = L.lib().abq_get_gemm_schedule()
    return {i: k for k, i in GEMM_SCHEDULES.items()}[v]


def autotune_linear(lin: "Linear", x: torch.Tensor, trials: int = 5,
                    out_dtype=torch.float16) -> AutotuneResult:
    """The GPU counterpart of the reference's tile search for a resident layer:
    time the engine's own schedules for this (M, N, K, p, q) -- the decode GEMV
    variants for M <= 8 (fused tensor-pipe kernel / bit-serial AND+popcount),
    the prefill GEMM schedules for M >= 9 (classic / stream-K) -- verify every
    schedule's output bit for bit against the first, leave the fastest selected
    (process-global, like abq_set_gemv_variant) and return the records
    (config_id = schedule name, tile fields 0).  Each schedule is timed as the
    serving path runs it: a CUDA graph of back-to-back calls."""
    if trials < 3:
        raise ValueError("autotune: need at least 3 trials")
    m = x.shape[0]
    old_v, old_s = L.lib().abq_get_gemv_variant(), L.lib().abq_get_gemm_schedule()
    if m <= 8:
        scheds = [("auto", lambda: (set_gemv_variant("auto"), set_gemm_schedule("auto"))),
                  ("popc", lambda: set_gemv_variant("popc"))]
    else:
        scheds = [("classic", lambda: (set_gemv_variant("auto"), set_gemm_schedule("classic"))),
                  ("stream_k", lambda: (set_gemv_variant("auto"), set_gemm_schedule("stream_k"))),
                  ("popc", lambda: set_gemv_variant("popc"))]
    out = torch.empty((m, lin.w.planes.rows), dtype=out_dtype, device=x.device)
    reference, records, best = None, [], 0
    try:
        for name, select in scheds:
            select()
            us = _time_graph_us(lambda: lin(x, out=out, check=False), trials)
            got = out.clone()
            if reference is None:
                reference = got
            elif not torch.equal(got, reference):
                raise Error(f"autotune: schedule {name} disagrees with the reference result")
            rec = BenchRecord(name, 0, 0, 0, 0, 0, lin.spec.planes(), lin.w.planes.planes, m,
                              lin.w.planes.rows, lin.k, us, tops_of(m, lin.w.planes.rows, lin.k, us))
            if records and us < records[best].median_us:
                best = len(records)
            records.append(rec)
    finally:
        L.lib().abq_set_gemv_variant(old_v)
        L.lib().abq_set_gemm_schedule(old_s)
    # leave the winner selected
    dict(scheds)[records[best].config_id]()
    return AutotuneResult(records[best].config_id, records)


def _gemm(fn, name, a: BitPlaneMatrix, bt: BitPlaneMatrix, tile, stats, dtype):
    out = torch.empty((a.rows, bt.rows), dtype=dtype, device=_dev())
    st = L.GemmStatsC(stats.block_tiles, stats.plane_pair_products) if stats is not None else None
    tc = tile.c() if tile is not None else None
    _check(fn(_ptr(a.data), a.planes, a.rows, a.cols, _ptr(bt.data), bt.planes, bt.rows, bt.cols,
              C.byref(tc) if tc is not None else None, _ptr(out),
              C.byref(st) if st is not None else None, _stream()))
    if stats is not None:
        stats.block_tiles, stats.plane_pair_products = st.block_tiles, st.plane_pair_products
    return out


def gemm_arbitrary(a: BitPlaneMatrix, bt: BitPlaneMatrix, tile: TileConfig,
                   stats: Optional[GemmStats] = None) -> torch.Tensor:
    """gemm_arbitrary  gemm.hpp:185-198 -> int32 M x N."""
    return _gemm(L.lib().abq_gemm_arbitrary, "gemm_arbitrary", a, bt, tile, stats, torch.int32)


def gemm_arbitrary_wide(a: BitPlaneMatrix, bt: BitPlaneMatrix, tile: TileConfig,
                        stats: Optional[GemmStats] = None) -> torch.Tensor:
    """gemm_arbitrary_wide  gemm.hpp:201-209 -> int64 M x N."""
    return _gemm(L.lib().abq_gemm_arbitrary_wide, "gemm_arbitrary_wide", a, bt, tile, stats,
                 torch.int64)


def gemm_naive(a: BitPlaneMatrix, bt: BitPlaneMatrix) -> torch.Tensor:
    """gemm_naive  gemm.hpp:213-231."""
    out = torch.empty((a.rows, bt.rows), dtype=torch.int32, device=_dev())
    _check(L.lib().abq_gemm_naive(_ptr(a.data), a.planes, a.rows, a.cols, _ptr(bt.data), bt.planes,
                                  bt.rows, bt.cols, _ptr(out), _stream()))
    return out


def zero_point_correct(acc: torch.Tensor, rowsum_a, colsum_b, z_a, z_b, k: int) -> torch.Tensor:
    """zero_point_correct  gemm.hpp:235-254 (int64 arithmetic, result in acc's dtype)."""
    m, n = acc.shape
    ra, cb = _to_dev(rowsum_a, torch.int64), _to_dev(colsum_b, torch.int64)
    za, zb = _to_dev(z_a, torch.int32), _to_dev(z_b, torch.int32)
    if ra.numel() != m or za.numel() != m:
        raise ShapeError("zero_point_correct: row-side vectors do not match")
    if cb.numel() != n or zb.numel() != n:
        raise ShapeError("zero_point_correct: col-side vectors do not match")
    acc = acc.contiguous()
    out = torch.empty_like(acc)
    fn = L.lib().abq_zero_point_correct_i32 if acc.dtype == torch.int32 else L.lib().abq_zero_point_correct_i64
    _check(fn(_ptr(acc), m, n, _ptr(ra), _ptr(cb), _ptr(za), _ptr(zb), k, _ptr(out), _stream()))
    return out


def code_rowsums(codes) -> torch.Tensor:
    """code_rowsums  gemm.hpp:256-261."""
    codes = _to_dev(codes, torch.uint8)
    out = torch.empty(codes.shape[0], dtype=torch.int64, device=_dev())
    _check(L.lib().abq_code_rowsums(_ptr(codes), codes.shape[0], codes.shape[1], _ptr(out), _stream()))
    return out


def plane_rowsums(m: BitPlaneMatrix) -> torch.Tensor:
    """code row sums recovered from the planes (= code_rowsums(unpack(m)))."""
    out = torch.empty(m.rows, dtype=torch.int64, device=_dev())
    _check(L.lib().abq_plane_rowsums(_ptr(m.data), m.planes, m.rows, m.cols, _ptr(out), _stream()))
    return out


# ---------------------------------------------------------------------------
# device-resident weights + fused linear (the engine hot path)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class PackedWeights:
    """Offline-packed weights resident in HBM: ABQP planes + per-channel
    scales / zero points + colsum_b.  The reference re-packs
    these on every quantized_linear call (gemm.hpp:274-278)."""
    planes: BitPlaneMatrix
    scales: torch.Tensor
    zero_points: torch.Tensor
    colsums: torch.Tensor
    per_tensor: bool
    frag: Optional[torch.Tensor] = None  # fragment-major copy for the tensor-pipe GEMV (M <= 8)
    tc: Optional[torch.Tensor] = None    # tcgen05-GEMM copy (M >= 9)

    @staticmethod
    def from_quantized(wt: QuantizedTensor, frag: bool = True, tc: bool = True) -> "PackedWeights":
        pm = bitpack(wt.codes, wt.spec.planes())
        return PackedWeights(pm, wt.scales.contiguous(), wt.zero_points.contiguous(),
                             plane_rowsums(pm), wt.spec.granularity == PER_TENSOR,
                             prepack_frag(pm) if frag else None, prepack_tc(pm) if tc else None)

    @staticmethod
    def from_planes(pm: BitPlaneMatrix, scales, zero_points, per_tensor=False,
                    frag: bool = True, tc: bool = True) -> "PackedWeights":
        return PackedWeights(pm, _to_dev(scales, torch.float64), _to_dev(zero_points, torch.int32),
                             plane_rowsums(pm), per_tensor, prepack_frag(pm) if frag else None,
                             prepack_tc(pm) if tc else None)

    def resident(self, layouts: str) -> "PackedWeights":
        """Serving copy that keeps ONE engine layout per regime in HBM and drops
        the ABQP planes: 'decode' = the GEMV layout (m <= 8), 'prefill' = the
        tcgen05 layout (any m), 'both' = the two.  Same bytes as the planes per
        layout (the full object holds planes + frag + tc = 3x).  The API-path
        entry points, shard() and copy() need the planes: call them on the
        full object."""
        if layouts not in ("decode", "prefill", "both"):
            raise ValueError("PackedWeights.resident: layouts must be 'decode', 'prefill' or 'both'")
        frag = self.frag if layouts in ("decode", "both") else None
        tc = self.tc if layouts in ("prefill", "both") else None
        if (layouts != "prefill" and frag is None) or (layouts != "decode" and tc is None):
            raise ValueError(f"PackedWeights.resident: the {layouts} layout was not built")
        pm = BitPlaneMatrix(self.planes.planes, self.planes.rows, self.planes.cols,
                            torch.empty(0, dtype=torch.int64, device=self.planes.data.device))
        return PackedWeights(pm, self.scales, self.zero_points, self.colsums, self.per_tensor, frag, tc)

    def resident_bytes(self) -> int:
        """HBM bytes of the packed weight layouts held (planes, frag, tc)."""
        return sum(t.numel() * t.element_size() for t in (self.planes.data, self.frag, self.tc) if t is not None)

    def c(self) -> L.WeightsC:
        return L.WeightsC(_ptr(self.planes.data) if self.planes.data.numel() else None,
                          self.planes.planes, self.planes.rows,
                          self.planes.cols, _ptr(self.scales), _ptr(self.zero_points),
                          _ptr(self.colsums), int(self.per_tensor),
                          _ptr(self.frag) if self.frag is not None else None,
                          _ptr(self.tc) if self.tc is not None else None)

    def copy(self) -> "PackedWeights":
        """Distinct HBM copy of the packed weights (same values)."""
        pm = BitPlaneMatrix(self.planes.planes, self.planes.rows, self.planes.cols,
                            self.planes.data.clone())
        return PackedWeights(pm, self.scales, self.zero_points, self.colsums, self.per_tensor,
                             self.frag.clone() if self.frag is not None else None,
                             self.tc.clone() if self.tc is not None else None)

    @staticmethod
    def concat(parts: List["PackedWeights"]) -> "PackedWeights":
        """Output-channel concatenation of layers that read the same input
        (fused q/k/v, gate/up): one engine launch computes all of them; column
        block j of the result is parts[j]'s output exactly (channels are
        independent)."""
        if not parts:
            raise ValueError("PackedWeights.concat: no parts")
        p0 = parts[0].planes
        if any(w.planes.planes != p0.planes or w.planes.cols != p0.cols for w in parts):
            raise ShapeError("PackedWeights.concat: parts differ in bit width or K")
        if any(w.per_tensor for w in parts):
            raise ValueError("PackedWeights.concat: per-channel weight scales required")
        pm = BitPlaneMatrix(p0.planes, sum(w.planes.rows for w in parts), p0.cols,
                            torch.cat([w.planes.data for w in parts], dim=1).contiguous())
        return PackedWeights(pm, torch.cat([w.scales for w in parts]), torch.cat([w.zero_points for w in parts]),
                             torch.cat([w.colsums for w in parts]), False,
                             prepack_frag(pm) if parts[0].frag is not None else None,
                             prepack_tc(pm) if parts[0].tc is not None else None)

    def shard(self, rank: int, world: int) -> "PackedWeights":
        """Column-parallel slice: output channels [rank*N/G, (rank+1)*N/G)
        (SURVEY.md 8e).  Each plane contributes a contiguous row range."""
        n = self.planes.rows
        lo, hi = n * rank // world, n * (rank + 1) // world
        pm = BitPlaneMatrix(self.planes.planes, hi - lo, self.planes.cols,
                            self.planes.data[:, lo:hi, :].contiguous())
        s = self.scales if self.per_tensor else self.scales[lo:hi].contiguous()
        z = self.zero_points if self.per_tensor else self.zero_points[lo:hi].contiguous()
        return PackedWeights(pm, s, z, self.colsums[lo:hi].contiguous(), self.per_tensor,
                             prepack_frag(pm) if self.frag is not None else None,
                             prepack_tc(pm) if self.tc is not None else None)


def prepack_frag(pm: BitPlaneMatrix) -> torch.Tensor:
    """K5: ABQP planes -> fragment-major planes for the tensor-pipe decode GEMV."""
    nbytes = L.lib().abq_weights_frag_bytes(pm.planes, pm.rows, pm.cols)
    frag = torch.empty(max(1, nbytes // 4), dtype=torch.int32, device=_dev())
    _check(L.lib().abq_weights_prepack(_ptr(pm.data), pm.planes, pm.rows, pm.cols, _ptr(frag), _stream()))
    return frag


def prepack_tc(pm: BitPlaneMatrix) -> torch.Tensor:
    """K5: ABQP planes -> tc planes for the tcgen05 prefill GEMM."""
    nbytes = L.lib().abq_weights_tc_bytes(pm.planes, pm.rows, pm.cols)
    tc = torch.empty(max(1, nbytes // 4), dtype=torch.int32, device=_dev())
    _check(L.lib().abq_weights_prepack_tc(_ptr(pm.data), pm.planes, pm.rows, pm.cols, _ptr(tc), _stream()))
    return tc


def set_gemv_variant(variant: str) -> None:
    """'auto' | 'popc' (AND+popcount on CUDA cores) | 'recomb' (planes on the int8 tensor pipe)."""
    _check(L.lib().abq_set_gemv_variant({"auto": 0, "popc": 1, "recomb": 2}[variant]))


_OUT = {torch.float16: L.ABQ_OUT_F16, torch.float64: L.ABQ_OUT_F64, torch.float32: L.ABQ_OUT_F32,
        torch.int64: L.ABQ_OUT_CORR_I64}


def linear_planes(a: BitPlaneMatrix, s_a, z_a, rowsum_a, w: PackedWeights, out_dtype=torch.float16,
                  a_per_tensor: bool = False, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Fused K2/K3 + K4 on packed activation planes."""
    if out is None:
        out = torch.empty((a.rows, w.planes.rows), dtype=out_dtype, device=_dev())
    act = L.ActC(_ptr(a.data), a.planes, a.rows, a.cols, _ptr(s_a), _ptr(z_a), _ptr(rowsum_a),
                 int(a_per_tensor))
    wc = w.c()
    _check(L.lib().abq_linear_planes(C.byref(act), C.byref(wc), _ptr(out), _OUT[out.dtype], _stream()))
    return out


def quant_pack_act(x: torch.Tensor, spec: QuantSpec):
    """K1: fused ReQuant + BitPacking of device activations (quantizer.hpp:146-213
    -> bitplane.hpp:47-64 -> gemm.hpp:256-261).  Returns (planes, scales,
    zero_points, rowsums)."""
    spec.validate()
    x = x.contiguous()
    m, k = x.shape
    p = spec.planes()
    groups = 1 if spec.granularity == PER_TENSOR else m
    planes = _empty_planes(p, m, k)
    sa = torch.empty(groups, dtype=torch.float64, device=x.device)
    za = torch.empty(groups, dtype=torch.int32, device=x.device)
    ra = torch.empty(m, dtype=torch.int64, device=x.device)
    cs = spec.c()
    _check(L.lib().abq_quant_pack_act(_ptr(x), _dtype_code(x), m, k, C.byref(cs), _ptr(planes),
                                      _ptr(sa), _ptr(za), _ptr(ra), None, None, _stream()))
    return BitPlaneMatrix(p, m, k, planes), sa, za, ra


class QAct:
    """Per-token quantized activations made by a producer op with the ReQuant
    fused in (rmsnorm_quant / silu_mul_quant), in the decode
    GEMV's code layout: codes + s_a / z_a / code row sums (quantizer.hpp:146-213
    applied to the producer's fp16 output).  Consumed by Linear(qact); one
    QAct feeds every projection that reads the same activations."""

    def __init__(self, m: int, k: int, spec: QuantSpec, device=None):
        spec.validate()
        if spec.granularity == PER_TENSOR:
            raise ValueError("QAct: the fused ReQuant is per token")
        dev = device or _dev()
        self.m, self.k, self.spec = m, k, spec
        nbytes = int(L.lib().abq_qact_codes_bytes(m, k))
        self.codes = torch.zeros(max(1, nbytes // 4), dtype=torch.int32, device=dev)
        self.scales = torch.empty(m, dtype=torch.float64, device=dev)
        self.zero_points = torch.empty(m, dtype=torch.int32, device=dev)
        self.rowsums = torch.empty(m, dtype=torch.int64, device=dev)
        self.err = torch.full((1,), -1, dtype=torch.int64, device=dev)
        self._c = L.QActC(_ptr(self.codes), _ptr(self.scales), _ptr(self.zero_points), _ptr(self.rowsums),
                          m, k, spec.bits)
        self._sc = spec.c()

    def c(self) -> L.QActC:
        return self._c

    def codes_matrix(self) -> np.ndarray:
        """u8 codes [m][k] decoded from the GEMV layout (tests / inspection)."""
        mt = 1 if self.m <= 1 else 2 if self.m <= 2 else 4 if self.m <= 4 else 8
        kpad = -(-self.k // 256) * 256
        words = self.codes.cpu().numpy().view(np.uint32)
        out = np.zeros((self.m, self.k), dtype=np.uint8)
        v = np.arange(self.k // 4)
        kb, rem = v >> 6, v & 63
        for t in range(self.m):
            tb, i = divmod(t, mt)
            idx = ((((kb * 8 + (rem >> 3)) * mt + i) * 4 + (rem & 3)) * 2) + ((rem >> 2) & 1)
            w = words[tb * mt * kpad // 4 + idx]
            out[t, :4 * len(v)] = np.stack([(w >> (8 * b)) & 0xFF for b in range(4)], 1).reshape(-1)
        return out

    def raise_if_nonfinite(self) -> None:
        v = int(self.err.item())
        if v != -1:
            raise ValueError(f"quantize: non-finite element at ({v // self.k},{v % self.k})")


def _producer_out(x: torch.Tensor, spec: QuantSpec, out: Optional[QAct]) -> QAct:
    m, k = x.shape
    if out is None:
        out = QAct(m, k, spec, x.device)
    elif (out.m, out.k) != (m, k) or out.spec.bits != spec.bits:
        raise ShapeError("QAct shape / bits differ from the producer input")
    return out


def rmsnorm_quant(x: torch.Tensor, gain: torch.Tensor, eps: float, spec: QuantSpec,
                  out: Optional[QAct] = None, y_out: Optional[torch.Tensor] = None,
                  check: bool = False) -> QAct:
    """LLaMA RMSNorm y = gain * fp16(x * rsqrt(mean(x^2) + eps)) (fp16 in/out)
    with the per-token ReQuant of y fused in (toyblock.hpp:257 -> 228-240).
    check=False: launch-only, a non-finite y is recorded in out.err."""
    if x.dtype != torch.float16 or gain.dtype != torch.float16 or x.dim() != 2 or not x.is_contiguous():
        raise ValueError("rmsnorm_quant: contiguous fp16 x [m][k] and fp16 gain [k] required")
    out = _producer_out(x, spec, out)
    if not check:
        out.err.fill_(-1)
    _check(L.lib().abq_rmsnorm_quant(_ptr(x), _ptr(gain.contiguous()), float(eps), x.shape[0], x.shape[1],
                                     C.byref(out._sc), _ptr(y_out) if y_out is not None else None,
                                     C.byref(out._c), None if check else _ptr(out.err), _stream()))
    return out


def silu_mul_quant(gate: torch.Tensor, up: torch.Tensor, spec: QuantSpec, out: Optional[QAct] = None,
                   y_out: Optional[torch.Tensor] = None, check: bool = False) -> QAct:
    """y = fp16(fp16(silu(gate)) * up) with the per-token ReQuant of y fused in
    (toyblock.hpp:274-275 -> 228-240)."""
    if gate.dtype != torch.float16 or up.dtype != torch.float16 or gate.shape != up.shape or gate.dim() != 2:
        raise ValueError("silu_mul_quant: fp16 gate / up of the same [m][k] shape required")
    gate, up = gate.contiguous(), up.contiguous()
    out = _producer_out(gate, spec, out)
    if not check:
        out.err.fill_(-1)
    _check(L.lib().abq_silu_mul_quant(_ptr(gate), _ptr(up), gate.shape[0], gate.shape[1], C.byref(out._sc),
                                      _ptr(y_out) if y_out is not None else None, C.byref(out._c),
                                      None if check else _ptr(out.err), _stream()))
    return out


class Linear:
    """One-call engine linear from fp16/fp32/fp64 activations: ReQuant +
    BitPacking (K1), plane GEMV/GEMM (K2/K3) and the fused epilogue (K4).
    Workspace is allocated once; call() is launch-only (no host sync) when
    check=False."""

    def __init__(self, weights: PackedWeights, act_spec: QuantSpec, max_m: int):
        act_spec.validate()
        self.w = weights
        self.spec = act_spec
        self.k = weights.planes.cols
        self.ws_bytes = L.lib().abq_linear_workspace_bytes(max_m, weights.planes.rows, self.k,
                                                           act_spec.planes())
        # zero-filled once; the engine leaves its cross-CTA accumulators zeroed
        self.ws = torch.zeros(self.ws_bytes, dtype=torch.uint8, device=_dev())
        self.err = torch.full((1,), -1, dtype=torch.int64, device=_dev())
        self.max_m = max_m
        self._wc = weights.c()
        self._sc = act_spec.c()

    def __call__(self, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                 out_dtype=torch.float16, check: bool = False) -> torch.Tensor:
        """y = quantized_linear(ReQuant(x), W) in one engine call.

        check=False (the serving default) is launch-only: a non-finite
        activation is recorded on the device and raised by the next
        raise_if_nonfinite(); check=True synchronises and raises at once
        (quantizer.hpp:155-160 semantics)."""
        if isinstance(x, QAct):
            return self._call_qact(x, out, out_dtype)
        if not isinstance(x, torch.Tensor) or x.dim() != 2:
            raise ShapeError("Linear: activations must be a 2-D tensor [M][K]")
        if x.dtype not in (torch.float16, torch.float32, torch.float64):
            raise ValueError(f"Linear: unsupported activation dtype {x.dtype}")
        if x.device != self.ws.device:
            raise ValueError(f"Linear: activations on {x.device}, weights on {self.ws.device}")
        if not x.is_contiguous():
            raise ValueError("Linear: activations must be contiguous (row stride K)")
        m = x.shape[0]
        if m > self.max_m:
            raise ValueError(f"Linear: m={m} exceeds max_m={self.max_m}")
        n = self.w.planes.rows
        if out is None:
            out = torch.empty((m, n), dtype=out_dtype, device=x.device)
        else:
            if out.dtype not in _OUT:
                raise ValueError(f"Linear: unsupported output dtype {out.dtype}")
            # (pinned host memory is accepted too: the epilogue writes it over PCIe)
            if tuple(out.shape) != (m, n) or not out.is_contiguous() or \
                    (out.device != x.device and not (out.device.type == "cpu" and out.is_pinned())):
                raise ShapeError(f"Linear: out must be a contiguous ({m}, {n}) tensor on {x.device} or pinned host")
        # x.shape[1] (not self.k): the C-ABI rejects an inner-dimension mismatch
        _check(L.lib().abq_linear(_ptr(x), _dtype_code(x), m, x.shape[1], C.byref(self._sc),
                                  C.byref(self._wc), _out_ptr(out), _OUT[out.dtype], _ptr(self.ws),
                                  self.ws_bytes, None if check else _ptr(self.err), _stream()))
        if not check:
            self._last_k = x.shape[1]
        return out

    def _call_qact(self, a: "QAct", out, out_dtype) -> torch.Tensor:
        """decode linear on producer-quantized activations (abq_linear_qact)"""
        if a.m > self.max_m:
            raise ValueError(f"Linear: m={a.m} exceeds max_m={self.max_m}")
        n = self.w.planes.rows
        if out is None:
            out = torch.empty((a.m, n), dtype=out_dtype, device=a.codes.device)
        elif out.dtype not in _OUT or tuple(out.shape) != (a.m, n) or not out.is_contiguous():
            raise ShapeError(f"Linear: out must be a contiguous ({a.m}, {n}) tensor of a supported dtype")
        _check(L.lib().abq_linear_qact(C.byref(a.c()), C.byref(self._wc), _ptr(out), _OUT[out.dtype], _stream()))
        return out

    def prefetch_next(self, nxt: Optional["Linear"]) -> "Linear":
        """Successor-layer hint (abq_weights.next): `nxt` is the linear the
        caller runs next on the same stream (a decode step's layer order is
        static).  In this layer's decode GEMV tail every CTA, once its own
        weights have landed, prefetches the first KB of its share of nxt's
        weights into L2, so HBM keeps streaming while this grid finishes and
        the next launch's CTAs start.  Results never depend on it; None clears."""
        self._next = nxt
        self._wc.next = C.addressof(nxt._wc) if nxt is not None else None
        return self

    def raise_if_nonfinite(self) -> None:
        """Synchronise and raise abq.ValueError if the last check=False call
        saw a non-finite activation (the report is reset by every call)."""
        v = int(self.err.item())
        if v != -1:
            k = getattr(self, "_last_k", self.k)
            raise ValueError(f"quantize: non-finite element at ({v // k},{v % k})")


class HostLinear:
    """End-to-end serving call on host buffers, without copy nodes: step()
    stages the pinned host activations into HBM with a kernel (abq_stage_in:
    PCIe loads issued at once, stores after the previous kernel completes) and
    runs the engine linear with its epilogue writing y straight into pinned
    host memory.  Both launches are programmatic-dependent, so consecutive
    steps overlap like a chain of layers (the next step's weights stream while
    the previous step finishes).  The caller synchronises before reading y_host."""

    def __init__(self, lin: "Linear", m: int, x_dtype=torch.float16, out_dtype=torch.float16):
        self.lin = lin
        k, n = lin.k, lin.w.planes.rows
        self.x_host = torch.empty((m, k), dtype=x_dtype, pin_memory=True)
        self.y_host = torch.empty((m, n), dtype=out_dtype, pin_memory=True)
        self.x_dev = torch.empty((m, k), dtype=x_dtype, device=_dev())
        self.h2d_bytes = self.x_host.numel() * self.x_host.element_size()
        self.d2h_bytes = self.y_host.numel() * self.y_host.element_size()
        if self.y_host.dtype not in _OUT:
            raise ValueError(f"HostLinear: unsupported output dtype {out_dtype}")
        # one C call per step (abq_linear_host) with its arguments bound once:
        # the step is otherwise host-bound on Python / ctypes overhead
        self._fn = L.lib().abq_linear_host
        self._stream = _stream()
        self._args = (self.x_host.data_ptr(), _dtype_code(self.x_dev), m, k, _ptr(self.x_dev), C.byref(lin._sc),
                      C.byref(lin._wc), self.y_host.data_ptr(), _OUT[self.y_host.dtype], _ptr(lin.ws), lin.ws_bytes,
                      _ptr(lin.err), self._stream)

    def step(self) -> torch.Tensor:
        """one step on the stream current at construction; raises on error"""
        st = self._fn(*self._args)
        if st:
            _check(st)
        return self.y_host


class GraphedHostLinear:
    """HostLinear's step captured as a CUDA graph: one replay per step runs the
    stage-in kernel (pinned x read over PCIe into HBM) and the engine linear
    whose epilogue writes y into pinned host memory -- no copy nodes, and no
    per-step host launch cost beyond one graph launch.  step() replays it; the
    caller synchronises before reading y_host."""

    def __init__(self, lin: "Linear", m: int, x_dtype=torch.float16, out_dtype=torch.float16):
        # the HostLinear is bound to the stream current at construction: build,
        # warm up and capture it on one side stream
        self._s = torch.cuda.Stream()
        self._s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self._s):
            self.host = HostLinear(lin, m, x_dtype, out_dtype)
            self.host.step()
        self._s.synchronize()
        self.x_host, self.y_host = self.host.x_host, self.host.y_host
        self.h2d_bytes, self.d2h_bytes = self.host.h2d_bytes, self.host.d2h_bytes
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self._s):
            self.host.step()

    def step(self) -> torch.Tensor:
        self.graph.replay()
        return self.y_host


class GraphedLinear:
    """Serving entry point: one decode/prefill step of a Linear captured as a
    CUDA graph together with its host I/O -- H2D of the activations from a
    pinned host buffer, the engine kernels, D2H of the fp16 result into a
    pinned host buffer.  step() replays it; the caller synchronises when it
    needs the result (e.g. via torch.cuda.current_stream().synchronize())."""

    def __init__(self, lin: Linear, m: int, x_dtype=torch.float16, out_dtype=torch.float16):
        self.lin = lin
        k, n = lin.k, lin.w.planes.rows
        self.x_host = torch.empty((m, k), dtype=x_dtype, pin_memory=True)
        self.y_host = torch.empty((m, n), dtype=out_dtype, pin_memory=True)
        self.x_dev = torch.empty((m, k), dtype=x_dtype, device=_dev())
        self.y_dev = torch.empty((m, n), dtype=out_dtype, device=_dev())
        self.h2d_bytes = self.x_host.numel() * self.x_host.element_size()
        self.d2h_bytes = self.y_host.numel() * self.y_host.element_size()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm up outside capture
            self._body()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._body()

    def _body(self):
        self.x_dev.copy_(self.x_host, non_blocking=True)
        self.lin(self.x_dev, out=self.y_dev, check=False)
        self.y_host.copy_(self.y_dev, non_blocking=True)

    def step(self) -> torch.Tensor:
        self.graph.replay()
        return self.y_host


def quantized_linear(act: QuantizedTensor, wt: QuantizedTensor,
                     stats: Optional[GemmStats] = None) -> torch.Tensor:
    """quantized_linear  gemm.hpp:266-307 -> float64 M x N, bit-identical to the
    reference (FP64 epilogue, same operation order)."""
    if act.cols() != wt.cols():
        raise ShapeError("quantized_linear: inner dimensions differ")
    p, q = act.spec.planes(), wt.spec.planes()
    a = bitpack(act.codes, p)
    w = PackedWeights.from_quantized(wt)
    rows_a = code_rowsums(act.codes)
    out = linear_planes(a, act.scales, act.zero_points, rows_a, w, torch.float64,
                        a_per_tensor=act.spec.granularity == PER_TENSOR)
    if stats is not None:
        t = default_tile(p, q)
        tiles = -(-act.rows() // t.BM) * -(-wt.rows() // t.BN)
        stats.block_tiles += tiles
        stats.plane_pair_products += tiles * p * q
    return out


def launch_count() -> int:
    return int(L.lib().abq_launch_count())
