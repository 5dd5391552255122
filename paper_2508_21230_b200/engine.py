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
from dataclasses import dataclass

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


def hole_slack(device: int) -> int:
    """Upper bound on unused record slots: every warp may leave one partly
    filled chunk (64 warps per SM is the hardware maximum)."""
    import torch

    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return sms * 64 * RECORD_CHUNK


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
        return DeviceData(device, cached[0], cached[1], hd.n_logical, n_dev, d_pad)
    dev = f"cuda:{device}"
    with torch.cuda.device(device):
        hv = torch.from_numpy(np.ascontiguousarray(hd.values))
        hn = torch.from_numpy(np.ascontiguousarray(hd.norms, dtype=np.float32))
        if n_dev == n_pad:
            values = hv.to(dev, non_blocking=True)
            norms = hn.to(dev, non_blocking=True)
        else:
            values = torch.zeros((n_dev, d_pad), dtype=torch.float16, device=dev)
            norms = torch.zeros(n_dev, dtype=torch.float32, device=dev)
            values[:n_pad].copy_(hv, non_blocking=True)
            norms[:n_pad].copy_(hn, non_blocking=True)
    return DeviceData(device, values, norms, hd.n_logical, n_dev, d_pad)


# Last exact count per problem, so repeated joins size their buffers once.
_count_memo: dict = {}
_memo_lock = threading.Lock()


def join_raw(dd: DeviceData, eps_sq: float, flags: int, rows, cols, records, capacity: int,
             count, stream) -> None:
    """One fasted_join launch (results stay on the device)."""
    st = _lib.load().fasted_join(dd.values.data_ptr(), dd.norms.data_ptr(), dd.n_logical,
                                 dd.n_dev, dd.d_pad, rows[0], rows[1], cols[0], cols[1],
                                 float(eps_sq), flags,
                                 records.data_ptr() if records is not None else None,
                                 capacity, count.data_ptr(), stream)
    _lib.check(st, "fasted_join")


def _estimate_capacity(dd: DeviceData, eps_sq: float, rows, cols, flags: int, stream) -> int:
    """Count-only join on a few evenly spaced row blocks -> capacity guess."""
    import torch

    r0, r1 = rows
    nblk = (r1 - r0) // BLOCK
    samples = min(nblk, 8)
    if samples == 0:
        return 0
    cnt = torch.zeros(2, dtype=torch.int64, device=f"cuda:{dd.device}")
    tot = 0
    for s in range(samples):
        b = r0 + (nblk * s // samples) * BLOCK
        join_raw(dd, eps_sq, flags | _lib.JOIN_COUNT, (b, b + BLOCK), cols, None, 0, cnt, stream)
        tot += int(cnt[0].item())
    return int(tot * nblk / samples * 1.25) + 65536


def join_device(dd: DeviceData, eps_sq: float, rows=None, cols=None, exact: bool = False,
                capacity: int | None = None, sort: bool = True) -> DeviceResult:
    """Run the join for rows x cols on dd.device; results stay on the device.
    With sort=False the raw 16-byte records are returned (res.records)."""
    import torch

    L = _lib.load()
    rows = rows or (0, dd.n_dev)
    cols = cols or (0, dd.n_dev)
    flags = _lib.JOIN_EXACT if exact else _lib.JOIN_TC
    dev = f"cuda:{dd.device}"
    with torch.cuda.device(dd.device):
        stream = torch.cuda.current_stream()
        sp = stream.cuda_stream
        key = (dd.n_dev, dd.d_pad, dd.n_logical, float(eps_sq), rows, cols, flags,
               dd.values.data_ptr())
        slack = hole_slack(dd.device)
        if capacity is None:
            with _memo_lock:
                capacity = _count_memo.get(key)
            if capacity is None:
                capacity = _estimate_capacity(dd, eps_sq, rows, cols, flags, sp)
            capacity += slack
        cnt = torch.zeros(2, dtype=torch.int64, device=dev)
        reruns = 0
        kernel_ms = 0.0
        while True:
            cap = max(int(capacity), 1)
            rec = torch.empty((cap, 4), dtype=torch.int32, device=dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            join_raw(dd, eps_sq, flags, rows, cols, rec, cap, cnt, sp)
            e1.record(stream)
            count, chunks = (int(v) for v in cnt.tolist())
            slots = chunks * RECORD_CHUNK
            kernel_ms += e0.elapsed_time(e1)
            if slots <= cap:
                break
            capacity = count + slack
            reruns += 1
        with _memo_lock:
            _count_memo[key] = count
        rec = rec[:slots]
        if not sort:
            return DeviceResult(None, None, None, count, kernel_ms, 0.0, reruns, slots, rec)
        oi = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        oj = torch.empty_like(oi)
        od = torch.empty(max(count, 1), dtype=torch.float32, device=dev)
        sort_ms = 0.0
        if count:
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            ws_bytes = L.fasted_sort_workspace_bytes(rows[1] - rows[0], dd.n_dev)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
            tj = torch.empty(count, dtype=torch.int32, device=dev)
            td = torch.empty(count, dtype=torch.float32, device=dev)
            s0.record(stream)
            _lib.check(L.fasted_sort_pairs(rec.data_ptr(), slots, rows[0], rows[1], dd.n_dev,
                                           oi.data_ptr(), oj.data_ptr(), od.data_ptr(),
                                           tj.data_ptr(), td.data_ptr(), ws.data_ptr(), ws_bytes,
                                           sp),
                       "fasted_sort_pairs")
            s1.record(stream)
            s1.synchronize()
            sort_ms = s0.elapsed_time(s1)
            del ws, tj, td
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


@dataclass
class JoinReport:
    kernel_seconds: float      # max over devices of the join kernel time
    merge_seconds: float       # sort + D2H (reference: merge)
    stage_seconds: float       # H2D upload
    wall_seconds: float
    per_device: list


def self_join_devices(hd, eps_sq: float, devices, exact: bool = False, row_range=None):
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
            dd = upload(hd, dev)
            torch.cuda.current_stream().synchronize()
            t_up = time.perf_counter() - t0
            res = join_device(dd, eps_sq, rows=parts[g], cols=(0, dd.n_dev), exact=exact)
            t1 = time.perf_counter()
            out = to_host(res)
            t_d2h = time.perf_counter() - t1
            return out, res, t_up, t_d2h

    if len(devices) == 1:
        results = [run(0)]
    else:
        with ThreadPoolExecutor(max_workers=len(devices)) as ex:
            results = list(ex.map(run, range(len(devices))))
    i = np.concatenate([r[0][0] for r in results])
    j = np.concatenate([r[0][1] for r in results])
    d = np.concatenate([r[0][2] for r in results])
    rep = JoinReport(
        kernel_seconds=max(r[1].kernel_ms for r in results) / 1e3,
        merge_seconds=max(r[1].sort_ms / 1e3 + r[3] for r in results),
        stage_seconds=max(r[2] for r in results),
        wall_seconds=time.perf_counter() - t_start,
        per_device=[{"device": devices[g], "rows": parts[g], "pairs": results[g][1].count,
                     "kernel_ms": results[g][1].kernel_ms, "sort_ms": results[g][1].sort_ms,
                     "reruns": results[g][1].reruns} for g in range(len(devices))],
    )
    return i, j, d, rep
