"""Device orchestration of the epsilon self-join (the B200 replacement of the
reference's worker threads + tile queue, tiling.py:307-351).

One host thread per GPU; each GPU holds a full FP16 copy of the dataset and
sweeps a contiguous range of 128-row blocks against every column, so the
path shards with no collective (north star (4)).  Per device:

    upload (H2D, skipped when to_half left the data resident)
    -> fasted_join       (tcgen05 kernel, or the bit-exact CUDA-core kernel)
                          16-byte pair records, unordered
    -> fasted_sort_pairs (canonical (i, j) order, SoA, on the device)
    -> D2H of (i, j, dist_sq)

Concatenating the devices' results in device order is globally sorted.
"""

from __future__ import annotations

import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ArgumentError

BLOCK = 128          # row-block granularity of the kernels and of the partitioner
RECORD_CHUNK = 256   # FASTED_RECORD_CHUNK in include/fasted.h
RECORD_BYTES = 16    # {i, j, dist_sq, 0}


@dataclass
class DeviceData:
    device: int
    values: "object"   # torch.float16 [n_dev, d_pad], n_dev % 128 == 0
    norms: "object"    # torch.float32 [n_dev]
    n_logical: int
    n_dev: int
    d_pad: int
    # upload_segmented: [(row_end, cuda event)] ascending -- rows [0, row_end)
    # are resident once the event completed (None: resident on the stream)
    ready: "object" = None
    # the host dataset's count memo (HalfDataset.count_memo): a fresh device
    # copy per call still finds the last exact count; a DeviceData made
    # without a HalfDataset keeps its own
    memo: dict = field(default_factory=dict)
    # (start, end) timing events around the H2D copy (None: no copy made)
    h2d: "object" = None

    def h2d_ms(self) -> float:
        """Device time of the upload (waits for it; 0 if nothing was copied)."""
        if self.h2d is None:
            return 0.0
        _poll(self.h2d[1])
        return self.h2d[0].elapsed_time(self.h2d[1])

    def wait_rows(self, stream, row_end: int) -> None:
        """Make `stream` wait until rows [0, row_end) are resident."""
        if self.ready is None:
            return
        for end, ev in self.ready:
            if end >= row_end:
                stream.wait_event(ev)
                return
        stream.wait_event(self.ready[-1][1])


@dataclass
class DeviceResult:
    i: "object"          # torch.int32 [count], canonical order (None if unsorted)
    j: "object"
    d: "object"
    count: int
    kernel_ms: float     # CUDA-event time of the join launch(es)
    sort_ms: float
    reruns: int
    slots: int           # record slots the kernel used (>= count; unused have i == 0)
    records: "object" = None   # torch.int32 [slots, 4] raw records (kept when unsorted)


def partition_rows(n_dev: int, parts: int) -> list:
    """Contiguous 128-row-block ranges, imbalance <= 1 block."""
    if parts < 1:
        raise ArgumentError("need at least one device")
    R = n_dev // BLOCK
    return [((R * g // parts) * BLOCK, (R * (g + 1) // parts) * BLOCK) for g in range(parts)]


def max_holes(device: int) -> int:
    """Upper bound on unused record slots: every warp may leave one partly
    filled chunk (64 warps per SM is the hardware maximum)."""
    import torch

    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return sms * 64 * RECORD_CHUNK


def hole_slack(device: int) -> int:
    """Record slots added to a count (estimate) when sizing a buffer."""
    return max_holes(device)


def upload(hd, device: int) -> DeviceData:
    """Device copy of a HalfDataset (row count padded to a multiple of 128)."""
    import torch

    _lib.require_device(device)
    n_pad, d_pad = hd.values.shape
    if d_pad % 16:
        raise ArgumentError(f"d_padded {d_pad} not a multiple of 16")
    n_dev = -(-n_pad // BLOCK) * BLOCK
    cached = hd.device_cache.get(device) if hasattr(hd, "device_cache") else None
    if cached is not None and tuple(cached[0].shape) == (n_pad, d_pad) and n_dev == n_pad:
        return DeviceData(device, cached[0], cached[1], hd.n_logical, n_dev, d_pad,
                          memo=_memo_of(hd))
    dev = f"cuda:{device}"
    with torch.cuda.device(device):
        hv = torch.from_numpy(np.ascontiguousarray(hd.values))
        hn = torch.from_numpy(np.ascontiguousarray(hd.norms, dtype=np.float32))
        cur = torch.cuda.current_stream()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if n_dev == n_pad:
            values = torch.empty((n_dev, d_pad), dtype=torch.float16, device=dev)
            norms = torch.empty(n_dev, dtype=torch.float32, device=dev)
        else:
            values = torch.zeros((n_dev, d_pad), dtype=torch.float16, device=dev)
            norms = torch.zeros(n_dev, dtype=torch.float32, device=dev)
        t0.record(cur)
        values[:n_pad].copy_(hv, non_blocking=True)
        norms[:n_pad].copy_(hn, non_blocking=True)
        t1.record(cur)
    return DeviceData(device, values, norms, hd.n_logical, n_dev, d_pad, memo=_memo_of(hd),
                      h2d=(t0, t1))


SEGMENT_MIN_BYTES = 256 << 20   # datasets below this upload in one piece
UPLOAD_SEGMENTS = 16


def upload_segmented(hd, device: int, segments: int = UPLOAD_SEGMENTS) -> DeviceData:
    """upload() in row segments on a copy stream, one event per segment
    (DeviceData.ready), so joins over the first rows can start while the
    rest is in flight.  Needs pinned host arrays (else: plain upload)."""
    import torch

    _lib.require_device(device)
    n_pad, d_pad = hd.values.shape
    n_dev = -(-n_pad // BLOCK) * BLOCK
    hv = torch.from_numpy(np.ascontiguousarray(hd.values)) if isinstance(hd.values, np.ndarray) \
        else hd.values
    cached = hd.device_cache.get(device) if hasattr(hd, "device_cache") else None
    if (segments <= 1 or hd.values.nbytes < SEGMENT_MIN_BYTES or n_dev != n_pad
            or not hv.is_pinned() or d_pad % 16 or cached is not None):
        return upload(hd, device)
    hn = torch.from_numpy(np.ascontiguousarray(hd.norms, dtype=np.float32)) \
        if isinstance(hd.norms, np.ndarray) else hd.norms
    dev = f"cuda:{device}"
    with torch.cuda.device(device):
        values = torch.empty((n_dev, d_pad), dtype=torch.float16, device=dev)
        norms = torch.empty(n_dev, dtype=torch.float32, device=dev)
        cur = torch.cuda.current_stream()
        copy = torch.cuda.Stream(device)
        copy.wait_stream(cur)          # the buffers above come from the current stream
        blocks = n_dev // BLOCK
        bounds = [BLOCK * (blocks * k // segments) for k in range(segments + 1)]
        ready = []
        t0 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(copy):
            t0.record(copy)
            for a, b in zip(bounds[:-1], bounds[1:]):
                if b <= a:
                    continue
                values[a:b].copy_(hv[a:b], non_blocking=True)
                norms[a:b].copy_(hn[a:b], non_blocking=True)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(copy)
                ready.append((b, ev))
        # the tensors were produced on `copy`: keep the allocator from reusing
        # them early when the caller frees them from another stream
        values.record_stream(copy)
        norms.record_stream(copy)
    return DeviceData(device, values, norms, hd.n_logical, n_dev, d_pad, ready,
                      memo=_memo_of(hd), h2d=(t0, ready[-1][1]))


def column_segments(dd: DeviceData, cols, first_rows_end: int) -> list:
    """Column launches for a row chunk while the dataset is still arriving:
    [(c0, c1, rows that must be resident)].  The first covers every column
    resident once the chunk's own rows are (the first upload segment ending
    at or after `first_rows_end`); the second takes the rest in one launch --
    it waits for the whole copy, which lands long before the first launch
    ends (C4: 35 ms of H2D against ~100 ms for the first launch).  Each
    launch may leave one partly filled 256-record run per warp, so the
    caller sizes the record buffer for len(result) launches."""
    if dd.ready is None:
        return [(cols[0], cols[1], cols[1])]
    first = next((end for end, _ in dd.ready if end >= first_rows_end), dd.ready[-1][0])
    first = min(max(first, cols[0]), cols[1])
    if first <= cols[0] or first >= cols[1]:
        return [(cols[0], cols[1], max(cols[1], first_rows_end))]
    return [(cols[0], first, max(first, first_rows_end)), (first, cols[1], dd.n_dev)]


def _poll(ev) -> None:
    """Wait for a CUDA event by polling.  Measured through self_join at
    1M x 960: a blocking cudaEventSynchronize / cudaStreamSynchronize returned
    10-1000 ms after the event completed on the GPU (its elapsed_time) in
    about one call of three, leaving the GPU idle; polling returns within
    ~0.2 ms every time."""
    while not ev.query():
        time.sleep(0.0002)


def _poll_stream(stream) -> None:
    import torch

    ev = torch.cuda.Event()
    ev.record(stream)
    _poll(ev)


def read_counts(cnt, stream=None) -> list:
    """Device int64 counters -> Python ints, ordered after `stream`'s work
    (the current stream by default), waiting by polling (see _poll)."""
    import torch

    st = stream if stream is not None else torch.cuda.current_stream(cnt.device)
    host = torch.empty(cnt.shape, dtype=cnt.dtype, pin_memory=True)
    with torch.cuda.stream(st):
        host.copy_(cnt, non_blocking=True)
    _poll_stream(st)
    return [int(v) for v in host.tolist()]


# Last exact count per problem (kept on the dataset, HalfDataset.count_memo),
# so repeated joins size their buffers once.
_memo_lock = threading.Lock()
MEMO_MAX = 64


def _memo_of(hd) -> dict:
    memo = getattr(hd, "count_memo", None)
    return memo if memo is not None else {}


def _memo_get(dd: DeviceData, key):
    with _memo_lock:
        return dd.memo.get(key)


def _memo_put(dd: DeviceData, key, count: int) -> None:
    with _memo_lock:
        if key not in dd.memo and len(dd.memo) >= MEMO_MAX:
            dd.memo.clear()
        dd.memo[key] = int(count)


def join_raw(dd: DeviceData, eps_sq: float, flags: int, rows, cols, records, capacity: int,
             count, stream, lib=None) -> None:
    """One fasted_join launch (results stay on the device).  `lib`: the
    library to call (default libfasted.so; the bit-identity tests pass
    _lib.load_experimental() to force other kernel forms)."""
    L = lib if lib is not None else _lib.load()
    st = L.fasted_join(dd.values.data_ptr(), dd.norms.data_ptr(), dd.n_logical,
                                 dd.n_dev, dd.d_pad, rows[0], rows[1], cols[0], cols[1],
                                 float(eps_sq), flags,
                                 records.data_ptr() if records is not None else None,
                                 capacity, count.data_ptr(), stream)
    _lib.check(st, "fasted_join", L)


def _estimate_capacity(dd: DeviceData, eps_sq: float, rows, cols, flags: int, stream,
                       lib=None) -> int:
    """Count-only join on a few evenly spaced row blocks -> capacity guess."""
    import torch

    r0, r1 = rows
    nblk = (r1 - r0) // BLOCK
    samples = min(nblk, 8)
    if samples == 0:
        return 0
    cnt = torch.zeros(2, dtype=torch.int64, device=f"cuda:{dd.device}")
    for s in range(samples):   # the sample blocks append into one count: one readback
        b = r0 + (nblk * s // samples) * BLOCK
        join_raw(dd, eps_sq, flags | _lib.JOIN_COUNT | (_lib.JOIN_APPEND if s else 0),
                 (b, b + BLOCK), cols, None, 0, cnt, stream, lib)
    tot = read_counts(cnt)[0]
    return int(tot * nblk / samples * 1.25) + 65536


def _sort_records(dd: DeviceData, rec, slots: int, count: int, rows, stream, out=None,
                  timed: bool = True, tmp=None, ws=None):
    """fasted_sort_pairs of `slots` raw records into canonical (i, j) SoA
    order on the device.  `out` = preallocated (i, j, d) tensors of length
    >= count, else allocated here.  Returns (i, j, d, sort_ms)."""
    import torch

    L = _lib.load()
    dev = f"cuda:{dd.device}"
    if out is None:
        oi = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        oj = torch.empty_like(oi)
        od = torch.empty(max(count, 1), dtype=torch.float32, device=dev)
    else:
        oi, oj, od = out
    sort_ms = 0.0
    if count:
        ws_bytes = L.fasted_sort_workspace_bytes(rows[1] - rows[0], dd.n_dev)
        if ws is None or ws.numel() < ws_bytes:
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        # scratch: the row-bucketed (j, dist_sq) pairs, 8 bytes per valid record
        if tmp is None or tmp.numel() < count:
            tjd = torch.empty(count, dtype=torch.int64, device=dev)
        else:
            tjd = tmp
        if timed:
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
        _lib.check(L.fasted_sort_pairs(rec.data_ptr(), slots, rows[0], rows[1], dd.n_dev,
                                       oi.data_ptr(), oj.data_ptr(), od.data_ptr(),
                                       tjd.data_ptr(), tjd.numel() * 8, ws.data_ptr(), ws.numel(),
                                       stream.cuda_stream),
                   "fasted_sort_pairs")
        if timed:
            s1.record(stream)
            s1.synchronize()
            sort_ms = s0.elapsed_time(s1)
        del ws, tjd   # stream-ordered reuse by the caching allocator is safe
    return oi, oj, od, sort_ms


def join_device(dd: DeviceData, eps_sq: float, rows=None, cols=None, exact: bool = False,
                capacity: int | None = None, sort: bool = True, flags: int = 0,
                lib=None) -> DeviceResult:
    """Run the join for rows x cols on dd.device; results stay on the device.
    With sort=False the raw 16-byte records are returned (res.records).
    `flags`: extra fasted_join flags (e.g. _lib.JOIN_SYMMETRIC); `lib`: see
    join_raw."""
    import torch

    L = _lib.load()
    rows = rows or (0, dd.n_dev)
    cols = cols or (0, dd.n_dev)
    flags |= _lib.JOIN_EXACT if exact else _lib.JOIN_TC
    dev = f"cuda:{dd.device}"
    with torch.cuda.device(dd.device):
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        key = (dd.n_dev, dd.d_pad, dd.n_logical, float(eps_sq), tuple(rows), tuple(cols), flags)
        slack = hole_slack(dd.device)
        if capacity is None:
            capacity = _memo_get(dd, key)
            if capacity is None:
                capacity = _estimate_capacity(dd, eps_sq, rows, cols,
                                              flags & ~_lib.JOIN_SYMMETRIC, sp, lib)
            capacity += slack
        if not exact:
            flags |= form_hints(capacity - slack, rows, cols)   # kernel-form hints only
        cnt = torch.zeros(2, dtype=torch.int64, device=dev)
        reruns = 0
        kernel_ms = 0.0
        while True:
            cap = max(int(capacity), 1)
            rec = torch.empty((cap, 4), dtype=torch.int32, device=dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            join_raw(dd, eps_sq, flags, rows, cols, rec, cap, cnt, sp, lib)
            e1.record(stream)
            count, chunks = read_counts(cnt, stream)
            slots = chunks * RECORD_CHUNK
            kernel_ms += e0.elapsed_time(e1)
            if slots <= cap:
                break
            capacity = count + slack
            reruns += 1
        _memo_put(dd, key, count)
        rec = rec[:slots]
        if not sort:
            return DeviceResult(None, None, None, count, kernel_ms, 0.0, reruns, slots, rec)
        oi, oj, od, sort_ms = _sort_records(dd, rec, slots, count, rows, stream)
        del rec
    return DeviceResult(oi[:count], oj[:count], od[:count], count, kernel_ms, sort_ms, reruns,
                        slots)


def to_host(res: DeviceResult):
    """D2H into pinned buffers; returns numpy (i uint32, j uint32, d float32)."""
    import torch

    if res.records is not None:          # unsorted raw records: drop unused slots
        raw = res.records.cpu().numpy()
        keep = raw[:, 0] != 0
        return (raw[keep, 0].view(np.uint32).copy(), raw[keep, 1].view(np.uint32).copy(),
                raw[keep, 2].view(np.float32).copy())
    n = res.count
    hi = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hj = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hd_ = torch.empty(n, dtype=torch.float32, pin_memory=True)
    if n:
        hi.copy_(res.i, non_blocking=True)
        hj.copy_(res.j, non_blocking=True)
        hd_.copy_(res.d, non_blocking=True)
        torch.cuda.current_stream(res.i.device).synchronize()
    return hi.numpy().view(np.uint32), hj.numpy().view(np.uint32), hd_.numpy()


class HostPairs:
    """Pinned host (i, j, dist_sq) arrays the pipeline appends into with
    async D2H copies; grows (rarely: the capacity starts from the sampled
    estimate) by reallocating and copying what is already there."""

    def __init__(self, capacity: int):
        self.cap = 0
        self.n = 0
        self.trace = None
        self.d2h_ms = 0.0
        self._alloc(max(int(capacity), 1))

    def _alloc(self, cap):
        import torch

        new = [torch.empty(cap, dtype=torch.int32, pin_memory=True),
               torch.empty(cap, dtype=torch.int32, pin_memory=True),
               torch.empty(cap, dtype=torch.float32, pin_memory=True)]
        if self.n:
            for a, b in zip(new, self.t):
                a[:self.n].copy_(b[:self.n])
        self.t = new
        self.cap = cap

    def reserve(self, extra: int, sync_streams=()):
        """Room for `extra` more pairs; waits for in-flight copies first if
        the buffers must move."""
        if self.n + extra <= self.cap:
            return
        for st in sync_streams:
            st.synchronize()
        self._alloc(max(self.n + extra, int(self.cap * 1.5)))

    def append_async(self, i, j, d, count: int, stream):
        """Enqueue the D2H of `count` pairs on `stream` (reserve() first)."""
        import torch

        if count:
            with torch.cuda.stream(stream):
                for dst, src in zip(self.t, (i, j, d)):
                    dst[self.n:self.n + count].copy_(src[:count], non_blocking=True)
        self.n += count

    def arrays(self):
        return (self.t[0][:self.n].numpy().view(np.uint32),
                self.t[1][:self.n].numpy().view(np.uint32), self.t[2][:self.n].numpy())


def plan_row_chunks(rows, est_records: int, budget_records: int, min_chunks: int = 1) -> list:
    """Split a 128-aligned row range into contiguous chunks whose expected
    record count fits `budget_records` (at least `min_chunks` when the range
    allows)."""
    r0, r1 = rows
    nblk = (r1 - r0) // BLOCK
    if nblk <= 0:
        return [rows]
    k = max(1, min_chunks, -(-int(est_records) // max(int(budget_records), 1)))
    k = min(k, nblk)
    return [(r0 + (nblk * c // k) * BLOCK, r0 + (nblk * (c + 1) // k) * BLOCK) for c in range(k)]


def taper_chunks(chunks: list) -> list:
    """Halve the first and the last of k >= 2 equal row chunks (k + 1 chunks,
    weights 1, 2, ..., 2, 1; no chunk grows): the first join starts once its
    smaller share of the dataset has landed (segmented upload) and the
    pipeline's exposed tail -- the last chunk's sort and D2H -- shrinks."""
    if len(chunks) < 2:
        return chunks
    r0, r1 = chunks[0][0], chunks[-1][1]
    nblk = (r1 - r0) // BLOCK
    k = len(chunks)
    w = [1] + [2] * (k - 1) + [1]
    if nblk < len(w):
        return chunks
    tot = sum(w)
    bounds = [0]
    acc = 0
    for x in w:
        acc += x
        bounds.append(nblk * acc // tot)
    return [(r0 + bounds[c] * BLOCK, r0 + bounds[c + 1] * BLOCK) for c in range(len(w))
            if bounds[c + 1] > bounds[c]]


# Chunking policy: a device streams its rows in chunks when the expected
# output is large -- bounded device memory (records + sorted copies of one
# chunk in flight, double buffered) and the sort + D2H of chunk c overlap
# the join of chunk c + 1.
PIPELINE_MIN_RECORDS = 1 << 22      # below this: one chunk (overlap not worth a launch)
LOW_OUTPUT_PER_ROW = 128            # FASTED_JOIN_LOW_OUTPUT hint threshold (pairs per row)
SPARSE_EXAMINED_PER_PAIR = 8192     # FASTED_JOIN_SPARSE: <= 1 pair per this many examined


def form_hints(expected_pairs: int, rows, cols) -> int:
    """Kernel-form hint flags for an expected output size (results are
    identical either way; include/fasted.h)."""
    nr = max(rows[1] - rows[0], 1)
    nc = max(cols[1] - cols[0], 1)
    f = 0
    if expected_pairs <= LOW_OUTPUT_PER_ROW * 1.25 * nr:
        f |= _lib.JOIN_LOW_OUTPUT
    if expected_pairs * SPARSE_EXAMINED_PER_PAIR <= nr * nc:
        f |= _lib.JOIN_SPARSE
    return f
TAPER_CHUNKS = False                # taper_chunks: C4 e2e 1.3205 s tapered (3 chunks) vs 1.3187 s (2)
PIPELINE_CHUNKS = 2                 # chunks for mid-size outputs (overlap; C4 e2e 1.304 vs 1.311 s at 4)
BYTES_PER_RECORD_IN_FLIGHT = 2 * 16 + 2 * 12 + 8   # raw x2, sorted x2, sort scratch


def _chunk_budget(device: int) -> int:
    import torch

    free, _ = torch.cuda.mem_get_info(device)
    return max(1 << 20, int(free * 0.5) // BYTES_PER_RECORD_IN_FLIGHT)


def stream_join(dd: DeviceData, eps_sq: float, rows, exact: bool, host: HostPairs,
                budget_records: int | None = None, symmetric: bool = False):
    """Row-chunked join -> sort -> D2H pipeline on one device, appending the
    canonical (i, j)-ordered pairs of `rows` x all columns to `host`.

    GPU stream order: join_0, join_1, sort_0, join_2, sort_1, ... : chunk
    c's count comes back on a side stream as soon as join c ends (while join
    c+1 runs), so sort c and join c+2 are queued before the GPU needs them;
    the D2H of chunk c runs on a copy stream beside join c + 2.  All buffers
    are allocated before the first launch.  Returns (kernel_ms, sort_ms,
    reruns, chunks).

    symmetric=True (tcgen05 only, rows = all rows): FASTED_JOIN_SYMMETRIC --
    only the tiles on or above the diagonal, each off-diagonal pair written
    in both orientations.  Mirrored records belong to any row, so the whole
    range is one chunk (one sort); if that does not fit the memory budget the
    full-matrix join runs instead (same pair set)."""
    import torch

    flags = _lib.JOIN_EXACT if exact else _lib.JOIN_TC
    cols = (0, dd.n_dev)
    if symmetric and (exact or tuple(rows) != cols):
        raise ArgumentError("symmetric join needs the tcgen05 path over all rows")
    dev = f"cuda:{dd.device}"
    with torch.cuda.device(dd.device):
        comp = torch.cuda.current_stream()
        copy = torch.cuda.Stream(dd.device)
        sp = comp.cuda_stream
        key = (dd.n_dev, dd.d_pad, dd.n_logical, float(eps_sq), tuple(rows), tuple(cols), flags)
        tr = {"estimate": 0.0, "reserve": 0.0, "wait_join": 0.0, "enqueue": 0.0, "drain": 0.0}
        tc0 = time.perf_counter()
        est = _memo_get(dd, key)
        if est is None:
            dd.wait_rows(comp, dd.n_dev)
            est = _estimate_capacity(dd, eps_sq, rows, cols, flags, sp)
        budget = budget_records or _chunk_budget(dd.device)
        if not exact:
            flags |= form_hints(est, rows, cols)   # kernel-form hints only (same results)
        min_chunks = PIPELINE_CHUNKS if est >= PIPELINE_MIN_RECORDS else 1
        chunks = plan_row_chunks(rows, est, budget, min_chunks)
        if TAPER_CHUNKS:
            chunks = taper_chunks(chunks)
        if symmetric:
            if est <= budget:
                chunks = [tuple(rows)]
                flags |= _lib.JOIN_SYMMETRIC
            else:
                symmetric = False
        tr["estimate"] = time.perf_counter() - tc0
        tc0 = time.perf_counter()
        host.reserve(int(est * 1.05) + 1024)
        tr["reserve"] += time.perf_counter() - tc0
        slack = hole_slack(dd.device)
        nrows = rows[1] - rows[0]

        def cap_for(ch):
            launches = len(column_segments(dd, cols, ch[1]))
            return int(est * (ch[1] - ch[0]) / max(nrows, 1) * 1.25) + slack * launches

        # Every buffer of the pipeline is allocated here, before the first
        # launch: a cudaMalloc issued while a join runs blocks the host until
        # the GPU drains (measured: 0.5 s GPU-idle gaps per call when the
        # sort outputs were allocated mid-pipeline).
        nbuf = 2 if len(chunks) > 1 else 1
        cap_max = max(cap_for(ch) for ch in chunks)
        out_cap = max(cap_max - slack, 1024)
        L = _lib.load()
        rec = [torch.empty((cap_max, 4), dtype=torch.int32, device=dev) for _ in range(nbuf)]
        if nbuf == 1:
            rec.append(rec[0])
        sorted_out = [(torch.empty(out_cap, dtype=torch.int32, device=dev),
                       torch.empty(out_cap, dtype=torch.int32, device=dev),
                       torch.empty(out_cap, dtype=torch.float32, device=dev))
                      for _ in range(nbuf)]
        if nbuf == 1:
            sorted_out.append(sorted_out[0])
        sort_tmp = torch.empty(out_cap, dtype=torch.int64, device=dev)
        max_rows = max(ch[1] - ch[0] for ch in chunks)
        sort_ws = torch.empty(max(L.fasted_sort_workspace_bytes(max_rows, dd.n_dev), 1),
                              dtype=torch.uint8, device=dev)
        cnt = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(2)]
        # counts come back on a side stream that waits only for ITS join: a
        # plain .tolist() would queue behind join c+1 on the compute stream
        # and leave the GPU idle until the host enqueued more work
        aux = torch.cuda.Stream(dd.device)
        cnt_h = torch.zeros((2, 2), dtype=torch.int64, pin_memory=True)
        cnt_ev = [None, None]
        d2h_done = [None, None]
        kernel_ms = 0.0
        sort_ms = 0.0
        reruns = 0
        total = 0
        tj = [None, None]
        sort_ev = []
        d2h_ev = []
        join_ev = []
        cnt_evs = []

        host_t0 = time.perf_counter()
        marks = []

        def mark(what):
            marks.append((what, round((time.perf_counter() - host_t0) * 1e3, 2)))

        def launch_join(c):
            b = c % 2
            mark("launch%d" % c)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            # while the dataset is still arriving (upload_segmented), chunk c
            # sweeps its columns segment by segment as they land, appending
            # to one record set; later chunks find everything resident
            segs = column_segments(dd, cols, chunks[c][1])
            if flags & _lib.JOIN_SYMMETRIC:    # one launch: rows == columns
                segs = [(cols[0], cols[1], dd.n_dev)]
            dd.wait_rows(comp, segs[0][2])
            e0.record(comp)
            for k, (c0, c1, need) in enumerate(segs):
                if k:
                    dd.wait_rows(comp, need)
                join_raw(dd, eps_sq, flags | (_lib.JOIN_APPEND if k else 0), chunks[c],
                         (c0, c1), rec[b], rec[b].shape[0], cnt[b], sp)
            e1.record(comp)
            tj[b] = (e0, e1)
            join_ev.append((c, e0, e1))
            aux.wait_event(e1)
            with torch.cuda.stream(aux):
                cnt_h[b].copy_(cnt[b], non_blocking=True)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(aux)
            cnt_ev[b] = ev
            cnt_evs.append((c, ev))
            mark("launched%d" % c)

        launch_join(0)
        if len(chunks) > 1:
            launch_join(1)
        for c in range(len(chunks)):
            b = c % 2
            e0, e1 = tj[b]
            tc0 = time.perf_counter()
            mark("wait%d" % c)
            _poll(cnt_ev[b])
            mark("synced%d" % c)
            count, used = (int(v) for v in cnt_h[b].tolist())
            tr["wait_join"] += time.perf_counter() - tc0
            tc0 = time.perf_counter()
            slots = used * RECORD_CHUNK
            kernel_ms += e0.elapsed_time(e1)
            if slots > rec[b].shape[0]:          # estimate too low: rerun this chunk
                reruns += 1
                dd.wait_rows(comp, dd.n_dev)
                comp.synchronize()
                rec[b] = torch.empty((count + max_holes(dd.device), 4), dtype=torch.int32,
                                     device=dev)
                if nbuf == 1:
                    rec[1 - b] = rec[b]
                r0 = torch.cuda.Event(enable_timing=True)
                r1 = torch.cuda.Event(enable_timing=True)
                r0.record(comp)
                join_raw(dd, eps_sq, flags, chunks[c], cols, rec[b], rec[b].shape[0], cnt[b], sp)
                r1.record(comp)
                r1.synchronize()
                kernel_ms += r0.elapsed_time(r1)
                count, used = (int(v) for v in cnt[b].tolist())
                slots = used * RECORD_CHUNK
            # sort_c lands behind join_{c+1} on the compute stream; its output
            # buffers are reused only after their previous D2H finished
            if d2h_done[b] is not None:
                comp.wait_event(d2h_done[b])
            out = sorted_out[b]
            if out[0].shape[0] < max(count, 1):      # estimate too low (rare)
                comp.synchronize()
                n_alloc = max(count, 1)
                out = (torch.empty(n_alloc, dtype=torch.int32, device=dev),
                       torch.empty(n_alloc, dtype=torch.int32, device=dev),
                       torch.empty(n_alloc, dtype=torch.float32, device=dev))
                sorted_out[b] = out
                if nbuf == 1:
                    sorted_out[1 - b] = out
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(comp)
            _sort_records(dd, rec[b], slots, count, chunks[c], comp, out=out, timed=False,
                          tmp=sort_tmp, ws=sort_ws)
            s1.record(comp)
            tr["enqueue"] += time.perf_counter() - tc0
            mark("sorted%d" % c)
            tc0 = time.perf_counter()
            host.reserve(count, sync_streams=(copy,))
            tr["reserve"] += time.perf_counter() - tc0
            copy.wait_event(s1)
            h0 = torch.cuda.Event(enable_timing=True)
            h0.record(copy)
            host.append_async(out[0], out[1], out[2], count, copy)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(copy)
            d2h_done[b] = ev
            d2h_ev.append((h0, ev))
            mark("d2h%d" % c)
            total += count
            # join c+2 reuses chunk c's record buffer: queued after sort c
            if c + 2 < len(chunks):
                launch_join(c + 2)
            sort_ev.append((s0, s1))
        tc0 = time.perf_counter()
        _poll_stream(copy)
        _poll_stream(comp)
        if dd.ready is not None:
            _poll(dd.ready[-1][1])
            dd.ready = None            # resident from here on
        tr["drain"] = time.perf_counter() - tc0
        sort_ms = sum(a.elapsed_time(b) for a, b in sort_ev)
        host.d2h_ms = sum(a.elapsed_time(b) for a, b in d2h_ev)
        host.trace = {k: round(v * 1e3, 2) for k, v in tr.items()}
        host.trace["host_marks"] = marks
        if join_ev:   # GPU timeline (ms from the first join start): gaps = GPU idle
            t0e = join_ev[0][1]
            host.trace["gpu_timeline"] = (
                [("join%d" % c, round(t0e.elapsed_time(a), 2), round(t0e.elapsed_time(b), 2))
                 for c, a, b in join_ev] +
                [("sort%d" % c, round(t0e.elapsed_time(a), 2), round(t0e.elapsed_time(b), 2))
                 for c, (a, b) in enumerate(sort_ev)] +
                [("count%d" % c, round(t0e.elapsed_time(e), 2)) for c, e in cnt_evs])
        _memo_put(dd, key, total)
    return kernel_ms, sort_ms, reruns, len(chunks)


@dataclass
class JoinReport:
    kernel_seconds: float      # max over devices of the join kernel time (CUDA events)
    merge_seconds: float       # pipeline time not hidden behind the join (sort + D2H tail)
    stage_seconds: float       # H2D upload, device time (CUDA events on the copy stream)
    wall_seconds: float
    per_device: list
    sort_seconds: float = 0.0  # max over devices of the device sort time
    d2h_seconds: float = 0.0   # max over devices of the result D2H device time


def self_join_devices(hd, eps_sq: float, devices, exact: bool = False, row_range=None,
                      symmetric: bool = False):
    """Row-block partition of `row_range` (default: all rows) across
    `devices`; returns (i, j, d, JoinReport)."""
    import torch

    for dev in set(devices):
        _lib.require_device(dev)
    t_start = time.perf_counter()
    n_dev = -(-hd.n_padded // BLOCK) * BLOCK
    r0, r1 = row_range if row_range is not None else (0, n_dev)
    parts = [(r0 + a, r0 + b) for a, b in partition_rows(r1 - r0, len(devices))]

    def run(g):
        dev = devices[g]
        with torch.cuda.device(dev):
            t0 = time.perf_counter()
            # segmented: the first row chunk starts on the first segments
            # while the rest of the dataset is still in flight
            dd = upload_segmented(hd, dev)
            if dd.ready is None:
                _poll_stream(torch.cuda.current_stream())
            t1 = time.perf_counter()
            host = HostPairs(1)
            kms, sms, reruns, nch = stream_join(dd, eps_sq, parts[g], exact, host,
                                                symmetric=symmetric)
            t_all = time.perf_counter() - t1
            return host, (kms, sms, reruns, nch), dd.h2d_ms() / 1e3, t_all

    if len(devices) == 1:
        results = [run(0)]
    else:
        with ThreadPoolExecutor(max_workers=len(devices)) as ex:
            results = list(ex.map(run, range(len(devices))))
    if len(results) == 1:
        # the pinned host buffers ARE the result arrays (no concatenation copy)
        i, j, d = results[0][0].arrays()
    else:
        # devices' shards in rank order = canonical order; one copy per device
        # part and array, in parallel (numpy releases the GIL for the memcpy)
        arrs = [r[0].arrays() for r in results]
        offs = np.cumsum([0] + [len(a[0]) for a in arrs])
        i = np.empty(offs[-1], np.uint32)
        j = np.empty(offs[-1], np.uint32)
        d = np.empty(offs[-1], np.float32)

        def place(job):
            g, k = job
            (i, j, d)[k][offs[g]:offs[g + 1]] = arrs[g][k]

        with ThreadPoolExecutor(max_workers=min(16, 3 * len(arrs))) as ex:
            list(ex.map(place, [(g, k) for g in range(len(arrs)) for k in range(3)]))
    rep = JoinReport(
        kernel_seconds=max(r[1][0] for r in results) / 1e3,
        merge_seconds=max(r[3] - r[1][0] / 1e3 for r in results),
        stage_seconds=max(r[2] for r in results),
        wall_seconds=time.perf_counter() - t_start,
        sort_seconds=max(r[1][1] for r in results) / 1e3,
        d2h_seconds=max(r[0].d2h_ms for r in results) / 1e3,
        per_device=[{"device": devices[g], "rows": parts[g], "pairs": results[g][0].n,
                     "h2d_ms": results[g][2] * 1e3, "d2h_ms": results[g][0].d2h_ms,
                     "kernel_ms": results[g][1][0], "sort_ms": results[g][1][1],
                     "reruns": results[g][1][2], "chunks": results[g][1][3],
                     "host_ms": getattr(results[g][0], "trace", None)}
                    for g in range(len(devices))],
    )
    return i, j, d, rep
