"""Device-resident, multi-stream entry points (the throughput path).

The reference API (fnt.py, cdc.py, aeq.py mirrors) moves numpy arrays per call.
For many channels / long streams the data stays in HBM instead:

* `CdcBank`   -- FNT-CDC over S streams x L samples in one launch, optionally
                 restricted to an output range (range shards with a halo) and
                 with the CDC->AEQ glue fused into its epilogue.
* `AeqBank`   -- S independent FNT-AEQ states, one warp per stream.
* `CdcAeqChain` -- the full per-link receiver chain of linksim.py:283-308 and
                 399-406: CDC on both polarizations (int8 in, fused requantized
                 int8 AEQ input and exact decimation statistics), the
                 decimation-phase decision, and the adaptive FNT-AEQ.

All tensors are torch CUDA tensors (plumbing); every compute step is a
libfntgpu kernel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .aeq import AeqConfig, aeq_params, mu_block_array
from .cdc import FntCdcEngine


def _t():
    return _lib.torch()


_TORCH2CODE = None


def _code(t) -> int:
    global _TORCH2CODE
    if _TORCH2CODE is None:
        tt = _t()
        _TORCH2CODE = {tt.int8: _lib.I8, tt.int16: _lib.I16, tt.int32: _lib.I32,
                       tt.int64: _lib.I64, tt.float64: _lib.F64, tt.complex128: _lib.C128}
    return _TORCH2CODE[t.dtype]


class CdcBank:
    """Launch wrapper around fntgpu_cdc64_process for one tap set."""

    def __init__(self, engine: FntCdcEngine):
        if not engine._fast():
            raise NotImplementedError("CdcBank runs the cdc64 plan")
        self.engine = engine
        self.inv_scale = 1.0 / engine.output_scale

    @property
    def taps(self):
        return self.engine.c_taps()  # current kernel selection (cdc.set_cdc_kernel)

    def _exact_requant(self, io, q_spec) -> None:
        """Integer requantization when (y * (1/output_scale)) * q_scale == y / 2^k up to
        rounding: q_scale is the engine's signal scale and its tap scale is 2^k
        (quantize_taps, cdc.py:80-86). The float64 results of the exact ties
        |y| = 2^(k-1) + j 2^k are evaluated here with the reference's expression."""
        import math
        ts = float(self.engine.tap_scale)
        k = int(round(math.log2(ts))) if ts > 0 else 0
        if (float(q_spec.scale) != float(self.engine.sig_spec.scale) or 2.0 ** k != ts
                or not 1 <= k <= 30 or q_spec.max_int > 127):
            return
        inv = self.inv_scale
        for j in range(int(q_spec.max_int) + 1):
            y = float((1 << (k - 1)) + j * (1 << k))
            v = (y * inv) * float(q_spec.scale)  # quantize_real on y * (1/output_scale)
            io.q_tie[j] = min(int(math.floor(abs(v) + 0.5)), int(q_spec.max_int))
        io.q_shift = k

    def run(self, xr, xi, *, length: int | None = None, x_first: int = 0,
            out_first: int = 0, out_count: int | None = None, yr=None, yi=None,
            qr=None, qi=None, q_spec=None, decim_acc=None, in_spec=None, in_clipped=None,
            stream=None) -> None:
        """xr, xi: (S, Lx) int8/int32/int64 device tensors holding global samples
        [x_first, x_first + Lx) of S streams of length `length`, or float64 front-end
        samples quantized on load with `in_spec` (quantize_real, fixedpoint.py:51-60;
        in_clipped: optional int64 device counter receiving the clip count). Outputs
        for the global range [out_first, out_first + out_count) go to yr/yi
        (S, out_count) (int16/int32/int64, or complex128 in yr) and/or the fused int8
        requantized planes qr/qi, and/or the decimation statistics decim_acc (S*8
        uint64)."""
        S, Lx = xr.shape
        length = Lx if length is None else length
        out_count = length - out_first if out_count is None else out_count
        io = _lib.CdcIO()
        io.n_streams = S
        io.in_dtype = _code(xr)
        io.xr, io.xi = xr.data_ptr(), xi.data_ptr()
        io.x_stride = xr.stride(0)
        io.x_first, io.x_count, io.length = x_first, Lx, length
        io.out_first, io.out_count = out_first, out_count
        io.out_dtype = _lib.NONE
        io.inv_scale = self.inv_scale
        if yr is not None:
            io.out_dtype = _code(yr)
            io.yr = yr.data_ptr()
            io.yi = yi.data_ptr() if yi is not None else None
            io.y_stride = yr.stride(0)
        io.q_shift = -1
        if qr is not None:
            io.qr, io.qi = qr.data_ptr(), qi.data_ptr()
            io.q_stride = qr.stride(0)
            io.q_scale = float(q_spec.scale)
            io.q_max = int(q_spec.max_int)
            self._exact_requant(io, q_spec)
        if decim_acc is not None:
            io.decim_acc = decim_acc.data_ptr()
        if io.in_dtype == _lib.F64:
            if in_spec is None:
                raise ValueError("float64 CDC input needs in_spec (the front-end QuantSpec)")
            io.in_scale = float(in_spec.scale)
            io.in_max = int(in_spec.max_int)
            io.in_clipped = in_clipped.data_ptr() if in_clipped is not None else None
        lib = _lib.load()
        st = _lib.vp(stream.cuda_stream) if stream is not None else _lib.stream_handle()
        _lib.check(lib.fntgpu_cdc64_process(C.byref(self.taps), C.byref(io), st), "cdc64_process")


#: Relative gap |m0 - m1| / max(m0, m1) between the two phase metrics below which the
#: device's decision (exact integer statistics, k_cdc.cu k_decim_phase) may differ from
#: the reference's float64 evaluation: its pairwise means and ratios carry a relative
#: error of at most a few 1e-14, so 1e-12 leaves a wide margin.
#: A NaN gap (an all-zero link: 0 / 0 in the reference) is treated as a tie as well.
PHASE_TIE_GUARD = 1e-12


def reference_phase(streams, sps: int = 2) -> int:
    """linksim._decimation_phase (linksim.py:249-260) in the reference's own float64
    numpy expression: the sampling phase minimizing sum over streams of
    mean|d|^4 / mean(|d|^2)^2, first minimum on ties (and phase 0 for NaN metrics)."""
    best, best_phase = None, 0
    for ph in range(sps):
        metric = 0.0
        for s in streams:
            d = s[ph::sps]
            p2 = np.mean(np.abs(d) ** 2)
            metric += np.mean(np.abs(d) ** 4) / (p2 * p2)
        if best is None or metric < best:
            best, best_phase = metric, ph
    return best_phase


def resolve_phase_ties(bank: "CdcBank", xr, xi, length: int, phase, gap,
                       guard: float | None = None) -> list[int]:
    """Links whose device phase decision is within float rounding of a tie get the
    reference's float64 decision: their CDC outputs (both polarizations, rows 2l and
    2l + 1 of xr / xi) are recomputed on the device and the metric is evaluated as
    linksim.py:249-260 does. Returns the resolved link indices (normally none).
    Synchronizes the current stream (one small device-to-host read of `gap`)."""
    t = _t()
    guard = PHASE_TIE_GUARD if guard is None else guard
    g = gap.cpu().numpy()
    idx = [int(i) for i in np.nonzero(~(g >= guard))[0]]
    if not idx:
        return idx
    inv = 1.0 / bank.engine.output_scale
    for l in idx:
        yr = t.empty((2, length), dtype=t.int32, device=xr.device)
        yi = t.empty_like(yr)
        bank.run(xr[2 * l:2 * l + 2], xi[2 * l:2 * l + 2], length=length, yr=yr, yi=yi)
        ar, ai = yr.cpu().numpy().astype(np.int64), yi.cpu().numpy().astype(np.int64)
        streams = [ar[p] * inv + 1j * (ai[p] * inv) for p in range(2)]  # cdc.py:177-180
        phase[l] = reference_phase(streams)
    return idx


def decimation_phase(acc, n_links: int, length: int, phase_out, gap_out=None, stream=None) -> None:
    io = _lib.DecimIO()
    io.n_links = n_links
    io.sps = 2
    io.acc = acc.data_ptr()
    io.length = length
    io.phase = phase_out.data_ptr()
    io.gap = gap_out.data_ptr() if gap_out is not None else None
    lib = _lib.load()
    st = _lib.vp(stream.cuda_stream) if stream is not None else _lib.stream_handle()
    _lib.check(lib.fntgpu_decim_phase(C.byref(io), st), "decim_phase")


class AeqBank:
    """S independent FNT-AEQ streams (device state), one warp each."""

    def __init__(self, config: AeqConfig, n_streams: int, forward: int | None = None):
        self.config = config
        self.n = n_streams
        self.prm = aeq_params(config, forward)
        self.state = _lib.zeros((n_streams * _lib.AEQ_STATE_BYTES,), np.uint8)
        self.reset()

    def reset(self, stream=None) -> None:
        lib = _lib.load()
        st = _lib.vp(stream.cuda_stream) if stream is not None else _lib.stream_handle()
        _lib.check(lib.fntgpu_aeq_init(_lib.ptr(self.state), self.n, C.byref(self.prm), st),
                   "aeq_init")

    def _io(self, n_blocks, adapt, mu_blocks, y, err):
        io = _lib.AeqIO()
        io.n_streams = self.n
        io.adapt = int(adapt)
        io.n_blocks = n_blocks
        io.mu_blocks = mu_blocks.data_ptr() if mu_blocks is not None else None
        io.y = y.data_ptr()
        io.y_stream_stride = y.stride(0)
        io.y_row_stride = y.stride(1)
        io.err = err.data_ptr() if err is not None else None
        io.err_stream_stride = err.stride(0) if err is not None else 0
        return io

    def run_planar(self, x, n_blocks: int, y, *, adapt=True, mu_blocks=None, err=None,
                   stream=None) -> None:
        """x: (S, 4, ld) int8/int32 device tensor; y: (S, 4, >=16 n_blocks) float64."""
        io = self._io(n_blocks, adapt, mu_blocks, y, err)
        io.in_mode = _lib.AEQ_IN_PLANAR
        io.in_dtype = _code(x)
        io.x = x.data_ptr()
        io.x_stream_stride = x.stride(0)
        io.x_row_stride = x.stride(1)
        self._launch(io, stream)

    def run_decim(self, qr, qi, phase, n_blocks: int, y, *, adapt=True, mu_blocks=None,
                  err=None, stream=None) -> None:
        """qr, qi: (2S, Lq) int8 requantized CDC planes (pol X = row 2s, pol Y = 2s+1);
        phase: (S,) int32 decimation phase per link."""
        io = self._io(n_blocks, adapt, mu_blocks, y, err)
        io.in_mode = _lib.AEQ_IN_DECIM
        io.in_dtype = _lib.I8
        io.qr, io.qi = qr.data_ptr(), qi.data_ptr()
        io.q_stride = qr.stride(0)
        io.phase = phase.data_ptr()
        self._launch(io, stream)

    def _launch(self, io, stream):
        lib = _lib.load()
        st = _lib.vp(stream.cuda_stream) if stream is not None else _lib.stream_handle()
        _lib.check(lib.fntgpu_aeq_process(_lib.ptr(self.state), C.byref(self.prm), C.byref(io), st),
                   "aeq_process")

    def read_state(self) -> list[_lib.AeqState]:
        raw = _lib.to_host(self.state).tobytes()
        sz = _lib.AEQ_STATE_BYTES
        return [_lib.AeqState.from_buffer_copy(raw[i * sz:(i + 1) * sz]) for i in range(self.n)]


class CdcAeqChain:
    """Receiver chain for n_links dual-polarization links of L samples each
    (linksim.py:283-308 + 399-406), all buffers preallocated in HBM.

    Inputs: xr, xi (2*n_links, L) int8 -- quantized front-end I/Q, row 2l = pol X
    and 2l+1 = pol Y of link l. Output: y (n_links, 4, 16*n_blocks) float64, the
    AEQ outputs [XI, XQ, YI, YQ]; err (n_links, n_blocks) the err_trace."""

    def __init__(self, engine: FntCdcEngine, aeq_config: AeqConfig, n_links: int, length: int,
                 sig_spec, mu_schedule=None, forward: int | None = None, keep_cdc_int=False,
                 tie_guard: bool = True):
        t = _t()
        self.tie_guard = tie_guard
        self.resolved: list[int] = []  # links whose phase the last run decided on the host
        dev = _lib.device()
        if length % 2:
            raise NotImplementedError("the chain runs 2 sps streams of even length")
        self.cdc = CdcBank(engine)
        self.n_links = n_links
        self.L = length
        self.sig_spec = sig_spec
        S = 2 * n_links
        # decimated length per phase is ceil((L - ph) / 2); both fit in Lq = ceil(L/2)
        self.n_sym = length // 2  # phase-1 length; phase 0 has ceil(L/2) >= this
        hop = aeq_config.l_taps
        self.n_blocks = (length - 1) // 2 // hop if length % 2 else (length // 2) // hop
        # q planes: padded to a multiple of 32 bytes so 32-byte loads stay in bounds
        lq = -(-length // 32) * 32 + 32
        self.qr = t.zeros((S, lq), dtype=t.int8, device=dev)
        self.qi = t.zeros((S, lq), dtype=t.int8, device=dev)
        self.acc = t.zeros((S * 8,), dtype=t.int64, device=dev)
        self.phase = t.zeros((n_links,), dtype=t.int32, device=dev)
        self.gap = t.zeros((n_links,), dtype=t.float64, device=dev)
        self.y = t.empty((n_links, 4, 16 * self.n_blocks), dtype=t.float64, device=dev)
        self.err = t.empty((n_links, max(self.n_blocks, 1)), dtype=t.float64, device=dev)
        self.yint = None
        if keep_cdc_int:
            self.yint = (t.empty((S, length), dtype=t.int16, device=dev),
                         t.empty((S, length), dtype=t.int16, device=dev))
        self.aeq = AeqBank(aeq_config, n_links, forward)
        mu = mu_block_array(self.n_blocks, hop, mu_schedule, aeq_config.mu)
        self.mu_blocks = t.from_numpy(mu).to(dev)

    def run(self, xr, xi, stream=None, reset=True) -> None:
        """One pass of the chain over the resident inputs (no host sync)."""
        if reset:
            self.aeq.reset(stream)
        self.acc.zero_()
        yr, yi = self.yint if self.yint is not None else (None, None)
        self.cdc.run(xr, xi, length=self.L, yr=yr, yi=yi, qr=self.qr, qi=self.qi,
                     q_spec=self.sig_spec, decim_acc=self.acc, stream=stream)
        decimation_phase(self.acc, self.n_links, self.L, self.phase, self.gap, stream=stream)
        if self.tie_guard:
            self.check_ties(xr, xi, stream)
        self.aeq.run_decim(self.qr, self.qi, self.phase, self.n_blocks, self.y, adapt=True,
                           mu_blocks=self.mu_blocks, err=self.err, stream=stream)

    def check_ties(self, xr, xi, stream=None) -> None:
        """Tie guard of the decimation phase (resolve_phase_ties); waits for the CDC."""
        t = _t()
        if stream is not None:
            with t.cuda.stream(stream):
                self.resolved = resolve_phase_ties(self.cdc, xr, xi, self.L, self.phase, self.gap)
        else:
            self.resolved = resolve_phase_ties(self.cdc, xr, xi, self.L, self.phase, self.gap)


class PipelinedChain:
    """The receiver chain as a steady-state pipeline over consecutive batches:
    the CDC (+ decimation phase) of batch k + 1 runs on its own CUDA stream while
    the FNT-AEQ of batch k runs, with two sets of intermediate buffers (requantized
    planes, statistics, phases). Every call is still one full pass of the chain
    over all links; outputs land in one y / err pair in call order (the AEQ
    launches are serialized on their stream). With few streams per SM the
    latency-bound AEQ leaves issue slots the CDC fills; with many, the CDC fills the
    AEQ's short last wave.

    Call `join()` before reading `y` / `err` of the last call."""

    def __init__(self, engine: FntCdcEngine, aeq_config: AeqConfig, n_links: int, length: int,
                 sig_spec, mu_schedule=None, forward: int | None = None):
        t = _t()
        dev = _lib.device()
        self.chains = [CdcAeqChain(engine, aeq_config, n_links, length, sig_spec, mu_schedule,
                                   forward) for _ in range(2)]
        b = self.chains[1]
        a = self.chains[0]
        # one AEQ state / output set: both buffer sets' AEQ runs share chain 0's
        b.aeq, b.y, b.err, b.mu_blocks = a.aeq, a.y, a.err, a.mu_blocks
        self.y, self.err, self.aeq = a.y, a.err, a.aeq
        self.s_cdc = t.cuda.Stream(device=dev)
        self.s_aeq = t.cuda.Stream(device=dev, priority=-1)  # the long-running launches first
        self.e_cdc = [t.cuda.Event() for _ in range(2)]
        self.e_aeq = [t.cuda.Event() for _ in range(2)]
        self.e_done = t.cuda.Event()
        self._calls = 0
        self.resolved: list[int] = []

    def __call__(self, xr, xi) -> None:
        t = _t()
        k = self._calls & 1
        ch = self.chains[k]
        caller = t.cuda.current_stream()
        self.s_cdc.wait_stream(caller)
        self.s_aeq.wait_stream(caller)
        if self._calls >= 2:  # the AEQ that last read this buffer set is done
            self.s_cdc.wait_event(self.e_aeq[k])
        with t.cuda.stream(self.s_cdc):
            ch.acc.zero_()
            ch.cdc.run(xr, xi, length=ch.L, qr=ch.qr, qi=ch.qi, q_spec=ch.sig_spec,
                       decim_acc=ch.acc, stream=self.s_cdc)
            decimation_phase(ch.acc, ch.n_links, ch.L, ch.phase, ch.gap, stream=self.s_cdc)
            ch.check_ties(xr, xi, self.s_cdc)
            self.resolved = ch.resolved
        self.e_cdc[k].record(self.s_cdc)
        self.s_aeq.wait_event(self.e_cdc[k])
        ch.aeq.reset(self.s_aeq)
        ch.aeq.run_decim(ch.qr, ch.qi, ch.phase, ch.n_blocks, ch.y, adapt=True,
                         mu_blocks=ch.mu_blocks, err=ch.err, stream=self.s_aeq)
        self.e_aeq[k].record(self.s_aeq)
        self.e_done.record(self.s_aeq)
        self._calls += 1

    def join(self, stream=None) -> None:
        """Make `stream` (default: the current stream) wait for the last call."""
        t = _t()
        (stream or t.cuda.current_stream()).wait_event(self.e_done)

    @property
    def phase(self):
        return self.chains[(self._calls - 1) & 1].phase


def _segments(total: int, parts: int, align: int) -> list[tuple[int, int]]:
    """Split [0, total) into <= parts contiguous ranges with boundaries on multiples
    of `align` (the last range takes the remainder)."""
    parts = max(1, min(parts, -(-total // align) if total else 1))
    step = -(-(-(-total // parts)) // align) * align
    out, a = [], 0
    while a < total:
        b = min(total, a + step)
        out.append((a, b))
        a = b
    return out or [(0, 0)]


class HostChain:
    """The receiver chain as a host-facing call: pinned host int8 I/Q in,
    float64 AEQ outputs and err_trace out (what a user of the reference's
    rx_frontend + run_single glue gets back), every call moving the data over
    PCIe. Used for the end-to-end measurement.

    The call is pipelined over three CUDA streams so the copies hide behind the
    kernels: the input arrives in `in_chunks` pieces and each piece's CDC output
    range (a range shard with its filter halo, sharding.py) starts as soon as the
    piece covering its halo has landed; the AEQ then runs in `aeq_segments` time
    segments (its state carries over between launches exactly as across
    FntAeq.process calls) and each segment's outputs stream back (strided 2-D
    copies) while the next segment computes. Consecutive calls overlap too: the
    next call's upload waits only for this call's CDC, its CDC for this call's
    AEQ, and each of its AEQ segments for the copy-out of the same segment. All
    work of a call is ordered after whatever the caller's stream had enqueued
    when the call was made; `join(stream)` makes a stream wait for the last call."""

    def __init__(self, engine: FntCdcEngine, aeq_config: AeqConfig, n_links: int, length: int,
                 sig_spec, mu_schedule=None, forward: int | None = None, in_chunks: int = 4,
                 aeq_segments: int = 8):
        t = _t()
        dev = _lib.device()
        self.chain = CdcAeqChain(engine, aeq_config, n_links, length, sig_spec, mu_schedule,
                                 forward)
        self.n_links, self.L = n_links, length
        self.dxr = t.empty((2 * n_links, length), dtype=t.int8, device=dev)
        self.dxi = t.empty_like(self.dxr)
        self.y = t.empty(tuple(self.chain.y.shape), dtype=t.float64, pin_memory=True)
        self.err = t.empty(tuple(self.chain.err.shape), dtype=t.float64, pin_memory=True)
        self.h2d_bytes = 2 * self.dxr.numel()
        self.d2h_bytes = 8 * (self.y.numel() + self.err.numel())
        # input pieces / CDC output ranges on 64-sample boundaries; AEQ block segments
        self.ranges = _segments(length, in_chunks, 64)
        self.segs = _segments(self.chain.n_blocks, aeq_segments, 1)
        self.s_in, self.s_cmp, self.s_out = (t.cuda.Stream(device=dev) for _ in range(3))
        E = lambda: t.cuda.Event()  # noqa: E731
        self.e_in = [E() for _ in self.ranges]
        self.e_cdc = E()
        self.e_aeq_done = E()
        self.e_seg = [E() for _ in self.segs]
        self.e_out = [E() for _ in self.segs]
        self.e_done = E()
        self._calls = 0

    def join(self, stream=None) -> None:
        """Make `stream` (default: the current stream) wait for the last call."""
        t = _t()
        (stream or t.cuda.current_stream()).wait_event(self.e_done)

    def __call__(self, xr_host, xi_host):
        t = _t()
        ch = self.chain
        lib = _lib.load()
        first = self._calls == 0
        caller = t.cuda.current_stream()
        for st in (self.s_in, self.s_cmp, self.s_out):
            st.wait_stream(caller)
        # -- upload (after the previous call's CDC has consumed the inputs)
        if not first:
            self.s_in.wait_event(self.e_cdc)
        for (a, b), ev in zip(self.ranges, self.e_in):
            _copy_rows(lib, self.dxr, xr_host, a, b, self.s_in)
            _copy_rows(lib, self.dxi, xi_host, a, b, self.s_in)
            ev.record(self.s_in)
        # -- CDC range shards (after the previous call's AEQ has consumed the q planes)
        if not first:
            self.s_cmp.wait_event(self.e_aeq_done)
        with t.cuda.stream(self.s_cmp):
            ch.aeq.reset(self.s_cmp)
            ch.acc.zero_()
            n_r = len(self.ranges)
            for j, (a, b) in enumerate(self.ranges):
                # output [a, b) reads inputs up to b + 48 (its blocks' halo): wait for the
                # piece holding them, and pass only the samples already landed (the
                # staging of a CTA's tail blocks past b treats the rest as zeros)
                jj = min(j + 1, n_r - 1)
                self.s_cmp.wait_event(self.e_in[jj])
                hi = self.ranges[jj][1]
                ch.cdc.run(self.dxr[:, :hi], self.dxi[:, :hi], length=self.L, out_first=a,
                           out_count=b - a, qr=ch.qr[:, a:], qi=ch.qi[:, a:],
                           q_spec=ch.sig_spec, decim_acc=ch.acc, stream=self.s_cmp)
            self.e_cdc.record(self.s_cmp)
            decimation_phase(ch.acc, ch.n_links, self.L, ch.phase, ch.gap, stream=self.s_cmp)
            if ch.tie_guard:
                ch.check_ties(self.dxr, self.dxi, self.s_cmp)
            # -- AEQ time segments; segment j's outputs may be overwritten only after the
            #    previous call copied them out
            for j, (b0, b1) in enumerate(self.segs):
                if not first:
                    self.s_cmp.wait_event(self.e_out[j])
                ch.aeq.run_decim(ch.qr[:, 32 * b0:], ch.qi[:, 32 * b0:], ch.phase, b1 - b0,
                                 ch.y[:, :, 16 * b0:], adapt=True, mu_blocks=ch.mu_blocks[b0:],
                                 err=ch.err[:, b0:], stream=self.s_cmp)
                self.e_seg[j].record(self.s_cmp)
            self.e_aeq_done.record(self.s_cmp)
        # -- copy-out per segment (y rows and err_trace entries of the segment's blocks)
        n4 = ch.y.shape[0] * ch.y.shape[1]
        row, erow = ch.y.shape[2] * 8, ch.err.shape[1] * 8
        so = _lib.vp(self.s_out.cuda_stream)
        for j, (b0, b1) in enumerate(self.segs):
            self.s_out.wait_event(self.e_seg[j])
            _lib.check(lib.fntgpu_copy2d_async(
                _lib.vp(self.y.data_ptr() + 128 * b0), row, _lib.vp(ch.y.data_ptr() + 128 * b0), row,
                128 * (b1 - b0), n4, so), "copy2d_async")
            _lib.check(lib.fntgpu_copy2d_async(
                _lib.vp(self.err.data_ptr() + 8 * b0), erow, _lib.vp(ch.err.data_ptr() + 8 * b0), erow,
                8 * (b1 - b0), ch.err.shape[0], so), "copy2d_async")
            self.e_out[j].record(self.s_out)
        self.e_done.record(self.s_out)
        self._calls += 1
        return self.y, self.err


def _copy_rows(lib, dev, host, a: int, b: int, stream) -> None:
    """host[:, a:b] -> dev[:, a:b] (int8 rows) as one strided 2-D copy."""
    rows, L = dev.shape
    _lib.check(lib.fntgpu_copy2d_async(_lib.vp(dev.data_ptr() + a), L, _lib.vp(host.data_ptr() + a),
                                       host.stride(0), b - a, rows, _lib.vp(stream.cuda_stream)),
               "copy2d_async")


class HostCdc:
    """FNT-CDC over host buffers: pinned int8 I/Q in -> H2D -> fntgpu_cdc64_process
    -> D2H int16 I/Q out (the decoded outputs of process_int, which fit int16
    within the engine's Eq. (5) budget). Used for the config-4 end-to-end number.

    Pipelined like HostChain: the samples move in `pieces` contiguous ranges; the
    CDC of output range j (a range shard with its filter halo) waits only for the
    input piece holding its halo, and its outputs stream back while range j + 1
    computes. The next call's upload of a piece waits for this call's CDC of it."""

    def __init__(self, engine: FntCdcEngine, n_streams: int, length: int, pieces: int = 8):
        t = _t()
        dev = _lib.device()
        if engine.budget.bound > 32767:
            raise NotImplementedError("int16 outputs need an Eq. (5) bound <= 32767")
        self.bank = CdcBank(engine)
        self.L = length
        self.dxr = t.empty((n_streams, length), dtype=t.int8, device=dev)
        self.dxi = t.empty_like(self.dxr)
        self.dyr = t.empty((n_streams, length), dtype=t.int16, device=dev)
        self.dyi = t.empty_like(self.dyr)
        self.yr = t.empty((n_streams, length), dtype=t.int16, pin_memory=True)
        self.yi = t.empty_like(self.yr, pin_memory=True)
        self.h2d_bytes = 2 * self.dxr.numel()
        self.d2h_bytes = 4 * self.dyr.numel()
        self.ranges = _segments(length, pieces, 64)
        self.s_in, self.s_cmp, self.s_out = (t.cuda.Stream(device=dev) for _ in range(3))
        E = lambda: t.cuda.Event()  # noqa: E731
        self.e_in = [E() for _ in self.ranges]
        self.e_cdc = [E() for _ in self.ranges]
        self.e_out = [E() for _ in self.ranges]
        self.e_done = E()
        self._calls = 0

    def join(self, stream=None) -> None:
        """Make `stream` (default: the current stream) wait for the last call."""
        t = _t()
        (stream or t.cuda.current_stream()).wait_event(self.e_done)

    def __call__(self, xr_host, xi_host):
        t = _t()
        lib = _lib.load()
        first = self._calls == 0
        caller = t.cuda.current_stream()
        for st in (self.s_in, self.s_cmp, self.s_out):
            st.wait_stream(caller)
        n_r = len(self.ranges)
        for j, (a, b) in enumerate(self.ranges):
            if not first:  # the previous call's CDC of ranges j - 1 and j read this piece
                self.s_in.wait_event(self.e_cdc[min(j + 1, n_r - 1)])
            _copy_rows(lib, self.dxr, xr_host, a, b, self.s_in)
            _copy_rows(lib, self.dxi, xi_host, a, b, self.s_in)
            self.e_in[j].record(self.s_in)
        for j, (a, b) in enumerate(self.ranges):
            jj = min(j + 1, n_r - 1)
            self.s_cmp.wait_event(self.e_in[jj])
            if not first:  # outputs of range j copied out by the previous call
                self.s_cmp.wait_event(self.e_out[j])
            hi = self.ranges[jj][1]  # only the samples already landed
            self.bank.run(self.dxr[:, :hi], self.dxi[:, :hi], length=self.L, out_first=a,
                          out_count=b - a, yr=self.dyr[:, a:], yi=self.dyi[:, a:],
                          stream=self.s_cmp)
            self.e_cdc[j].record(self.s_cmp)
        so = _lib.vp(self.s_out.cuda_stream)
        rows, pitch = self.dyr.shape[0], self.dyr.stride(0) * 2
        for j, (a, b) in enumerate(self.ranges):
            self.s_out.wait_event(self.e_cdc[j])
            for h, d in ((self.yr, self.dyr), (self.yi, self.dyi)):
                _lib.check(lib.fntgpu_copy2d_async(_lib.vp(h.data_ptr() + 2 * a), pitch,
                                                   _lib.vp(d.data_ptr() + 2 * a), pitch,
                                                   2 * (b - a), rows, so), "copy2d_async")
            self.e_out[j].record(self.s_out)
        self.e_done.record(self.s_out)
        self._calls += 1
        return self.yr, self.yi
