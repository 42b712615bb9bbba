#!/usr/bin/env python
"""Benchmark of the MoDM cache-retrieval hot path on B200 (one JSON line on rank 0).

Metric (BASELINE.json): cache lookups/sec at a 100k-entry cache; % of the
HBM / tensor roofline.  Default workload = BASELINE config 2: 100,000
entries x 768 dims, batch-1 lookups, one FIFO insert per request.  A step is
one lookup batch + its insert.  Config 3 (100k x 1024, batch 256) is measured
in the same run and reported under "c3".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value  = device time of K steps with inputs already in HBM (CUDA events on the
         library's stream, L2 flushed between steps, max over ranks);
e2e    = the same steps through the public API (SemanticCache.retrieve + add)
         from host buffers: H2D of the query and the inserted row and D2H of
         the decision are inside the timed region.
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK, TC_FALLBACK = 6650.0, 1590.0
METRIC = "cache lookups/sec at 100k-entry cache (batch 1 and 256); % of HBM/tensor roofline"
DATA = "synthetic clustered unit embeddings (reference generator model, spread 0.0554*sqrt(384/D), calibrated beta)"
C2_CONFIG = {"workload": "C2: 100k-entry FIFO cache, 768-dim, batch-1 lookup + FIFO insert per request",
             "entries": 100_000, "dim": 768, "batch": 1}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return HBM_FALLBACK, TC_FALLBACK, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self._wait_lines(1, 5.0)  # sampling is live before the timed region starts
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _wait_lines(self, n, timeout):
        t0 = time.time()
        while len(self.lines) < n and time.time() - t0 < timeout and self.proc and self.proc.poll() is None:
            time.sleep(0.005)

    def __exit__(self, *a):
        if self.proc:
            self._wait_lines(len(self.lines) + 1, 1.0)  # one sample after the timed region ends
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- workloads
def make_workload(dim: int, n_entries: int, n_queries: int, seed: int = 17):
    from paper_2503_11972_b200.workload import ClusteredWorkload

    wl = ClusteredWorkload(dim, n_clusters=512, seed=seed)
    rows = wl.cache_rows(n_entries)
    Q = wl.queries(n_queries)
    new_rows = wl.images(Q)
    return rows, Q, new_rows


def cpu_baseline(rows, Q, new_rows, insert: bool, seconds: float = 12.0, batch: int = 1):
    """The oracle port (float64 numpy/OpenBLAS, all host threads) timed on a bounded sample."""
    from oracle.retrieval import OracleCache, OracleEntry, OracleTable, blas_info

    n, dim = rows.shape
    o = OracleCache(n, dim)
    for i, v in enumerate(rows):
        o.insert(OracleEntry(f"e{i}", v, "large", i, 0.0))
    t = OracleTable()
    done = 0
    seq = n
    o.retrieve(Q[0], t)  # warm-up
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds and done < len(Q):
        for b in range(batch):  # the reference has no batch API: B sequential retrieves
            o.retrieve(Q[(done + b) % len(Q)], t)
        if insert:
            o.insert(OracleEntry(f"n{seq}", new_rows[done % len(new_rows)], "large", seq, 0.0))
            seq += 1
        done += batch
    dt = time.perf_counter() - t0
    threads = blas_threads()
    one = None
    try:  # the same path pinned to one BLAS thread, on a shorter sample
        from threadpoolctl import threadpool_limits

        with threadpool_limits(1, user_api="blas"):
            d1, t1 = 0, time.perf_counter()
            while time.perf_counter() - t1 < max(1.0, seconds / 4) and d1 < len(Q):
                o.retrieve(Q[d1 % len(Q)], t)
                d1 += 1
            one = d1 / (time.perf_counter() - t1)
    except Exception:
        pass
    return {
        "value": done / dt, "unit": "lookups/s", "cores": threads or os.cpu_count(), "kind": "port",
        "blas_threads": threads, "value_1thread": one,
        "sample": f"{done} sequential retrieve{'+insert' if insert else ''} calls on a {n}x{dim} float64 "
                  f"cache ({dt:.1f} s); {blas_info()}; host cpu_count={os.cpu_count()}",
    }


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((d.get("num_threads") or 0) for d in threadpool_info() if d.get("user_api") == "blas") or None
    except Exception:
        return None


# --------------------------------------------------------------------------- our arm
def run_config(name, dim, n_entries, B, steps, warmup, insert, flush_bytes, pk, device=0, n_rot=4, dist=None,
               e2e_steps=None):
    """One BASELINE config on one GPU.

    value: `steps` back-to-back lookup steps (B queries + the step's FIFO insert)
    rotating over n_rot caches of this shape with the same contents, whose scan
    copies together exceed L2 — every step streams its cache from HBM — timed
    by one pair of CUDA events around the whole run (mc_profile_rotate).  A
    per-step cross-check with events around each step and a 256 MiB L2 flush
    between steps (outside the events) is reported under "profile".
    """
    from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable, _native

    total = warmup + steps
    e2e_steps = max(steps, e2e_steps or steps)  # the public-API leg: enough requests for a stable rate
    n_q = total + (max(warmup, 200) if B == 1 else warmup) + 2 * e2e_steps + 8
    rows, Q, new_rows = make_workload(dim, n_entries, n_q * B)
    cache = SemanticCache(capacity=n_entries, dim=dim, device=device)
    cache.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n_entries))  # one device append
    table = ThresholdTable.default()
    cache.ring.set_table(table.pairs, table.total_steps)
    extra = []
    for _ in range(n_rot - 1):
        r = _native.DeviceRing(n_entries, dim, device)
        r.append(rows)
        r.set_table(table.pairs, table.total_steps)
        extra.append(r)
    rings = [cache.ring] + extra

    qd = Q[: total * B].reshape(total, B, dim)
    rd = new_rows[:total] if insert else None
    n_wrep = max(1, -(-50 // warmup))  # at least 50 untimed warm-up steps (W of them per pass)
    for _ in range(n_wrep):
        _native.DeviceRing.profile_rotate(rings, qd[:warmup], None if rd is None else rd[:warmup], warmup)
    if dist:
        dist.barrier()  # every rank enters the timed region together
    with ClockSampler(device) as clk:
        rot = _native.DeviceRing.profile_rotate(rings, qd[warmup:], None if rd is None else rd[warmup:], steps)
    if dist:  # the job's time is the slowest rank's
        rot["step_ms"] = dist.max_over_ranks(rot["step_ms"])
    # per-step cross-check: events around each step, L2 flushed between steps
    n_chk = min(steps, 200)
    prof = cache.ring.profile_steps(qd[warmup:warmup + n_chk], None if rd is None else rd[warmup:warmup + n_chk],
                                    n_chk, flush_bytes)
    for r in extra:
        r.close()
    # keep host metadata in step with ring 0 (it received every n_rot-th insert of each rotation call,
    # then the cross-check's inserts)
    if insert:
        idx = [i for i in range(warmup) if i % n_rot == 0] * n_wrep + [warmup + i for i in range(steps) if i % n_rot == 0]
        idx += [warmup + i for i in range(n_chk)]
        for i in idx:
            cache._store.append(CacheEntry(f"p{i}", new_rows[i], "large", cache._next_seq, 0.0))
            cache._next_seq += 1
            while len(cache._store) > cache.capacity:
                cache._store.popleft()
    assert len(cache._store) == len(cache.ring)
    step_ms = rot["step_ms"]
    value = (dist.world if dist else 1) * B / (step_ms * 1e-3)  # units all ranks processed / the job's time

    # e2e: public API from host buffers
    Qe = Q[total * B:].reshape(-1, B, dim)
    re = new_rows[total:]
    launches0 = cache.ring.stats()["kernel_launches"]
    t_base = 1000.0

    def run_e2e(first, count, tag, pipelined):
        """`count` requests through the public API.  B = 1: each request is its lookup and its FIFO
        insert, the insert staged while the scan runs (retrieve_async: the lookup sees the cache
        as retrieve() would; the insert only affects later lookups).  Pipelined: request i+1 is
        submitted before request i's answer is read (up to three lookups in flight, the API's limit), so
        the host's work overlaps the device's; the answers are those of the sequential loop."""
        prev = None
        ahead = collections.deque()  # batch 1, pipelined: up to three lookups in flight
        for i in range(first, first + count):
            if B == 1:
                pend = cache.retrieve_async(Qe[i][0], table)
                if insert:
                    cache.add(f"{tag}{i}", re[i], "large", t_base + i)
                if pipelined:
                    ahead.append(pend)
                    if len(ahead) == 3:
                        ahead.popleft().result()
                else:
                    pend.result()
            elif pipelined:  # batch i+1 uploaded and scanned while the host reads batch i's answers
                pend = cache.retrieve_batch_async(Qe[i], table)
                if insert:
                    cache.add(f"{tag}{i}", re[i], "large", t_base + i)
                if prev is not None:
                    int(prev.result().hit.sum())  # answers read back as arrays (objects build on access)
                prev = pend
            else:
                res = cache.retrieve_batch(Qe[i], table)
                int(res.hit.sum())  # the answers read back as arrays (result objects build on access)
                if insert:
                    cache.add(f"{tag}{i}", re[i], "large", t_base + i)
        while ahead:
            ahead.popleft().result()
        if prev is not None:
            r = prev.result()
            if B > 1:
                int(r.hit.sum())

    def timed_e2e(first, count, tag, pipelined):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        run_e2e(first, count, tag, pipelined)
        dt = time.perf_counter() - t0
        return dist.max_over_ranks(dt) if dist else dt

    if B > 4:  # batched queries come from one page-locked array: one DMA per batch, no staging copy
        cache.register_host_buffer(Q)
    n_warm = max(warmup, 200 if B == 1 else warmup)
    run_e2e(0, n_warm, "w", True)
    n_ranks = dist.world if dist else 1
    e2e_s = timed_e2e(n_warm, e2e_steps, "s", True)
    seq_s = timed_e2e(n_warm + e2e_steps, e2e_steps, "q", False)
    e2e_launches = (cache.ring.stats()["kernel_launches"] - launches0) / (n_warm + 2 * e2e_steps)
    e2e = {
        "value": n_ranks * B * e2e_steps / e2e_s, "unit": "lookups/s", "requests": e2e_steps,
        "latency_us": 1e6 * e2e_s / e2e_steps,
        "h2d_bytes_per_step": B * dim * 8 + (dim * 8 if insert else 0),
        "d2h_bytes_per_step": B * 24,
        "kernel_launches_per_step": e2e_launches,
        "mode": ("pipelined: retrieve_async of requests i+1 and i+2 before .result() of request i (three lookups "
                 "in flight)"
                 if B == 1 else "pipelined: retrieve_batch_async of batch i+1 before .result() of batch i"),
    }
    if B > 4:
        cache.unregister_host_buffer(Q)
        e2e["mode"] += "; queries taken from a page-locked array (SemanticCache.register_host_buffer)"
    if seq_s is not None:
        e2e["sequential"] = {"value": n_ranks * B * e2e_steps / seq_s, "unit": "lookups/s",
                             "latency_us": 1e6 * seq_s / e2e_steps,
                             "mode": ("one request at a time: retrieve_async, add, .result()" if B == 1
                                      else "one batch at a time: retrieve_batch")}
    st = cache.ring.stats()
    roof = roofline(st, n_entries, dim, B, step_ms, rot, prof, n_rot, pk, cfg=name)
    out = {
        "value": value, "ms_per_step": step_ms, "e2e": e2e, "roofline": roof, "clocks": clk.summary(),
        "gpu_launches": rot["launches_per_step"] * steps,
        "stats": st,
        "profile": dict(prof, rotation={"caches": n_rot, **rot}, untimed_warmup_steps=n_wrep * warmup,
                        per_step_check="events around each step, 256 MiB L2 flush between steps (outside the events)"),
        "rows": rows, "Q": Q, "new_rows": new_rows,
    }
    cache.close()
    return out


def run_generated(label, workload, dim, n_entries, B, steps, warmup, flush_bytes, pk, device=0):
    """A 1M-10M entry cache generated on the device (f4), `steps` back-to-back B-query lookups
    (the full decision epilogue in every launch), device-timed like C2's value.  The cache alone
    exceeds L2, so every step streams it from HBM without rotation."""
    from paper_2503_11972_b200 import ThresholdTable, _native
    from paper_2503_11972_b200.workload import GeneratedWorkload

    wl = GeneratedWorkload(dim, n_clusters=max(512, n_entries // 200), seed=17)
    ring = _native.DeviceRing(n_entries, dim, device)
    t0 = time.perf_counter()
    wl.fill(ring, n_entries)
    gen_s = time.perf_counter() - t0
    table = ThresholdTable.default()
    ring.set_table(table.pairs, table.total_steps)
    Q = wl.queries((warmup + steps) * B).reshape(warmup + steps, B, dim)
    _native.DeviceRing.profile_rotate([ring], Q[:warmup], None, warmup)
    with ClockSampler(device) as clk:
        rot = _native.DeviceRing.profile_rotate([ring], Q[warmup:], None, steps)
    prof = ring.profile_steps(Q[warmup:warmup + min(steps, 20)], None, min(steps, 20), flush_bytes)
    st = ring.stats()
    roof = roofline(st, n_entries, dim, B, rot["step_ms"], rot, prof, 1, pk)
    ring.close()
    return {"workload": label, "entries": n_entries, "dim": dim, "batch": B,
            "value": B / (rot["step_ms"] * 1e-3), "unit": "lookups/s", "ms_per_step": rot["step_ms"],
            "roofline": roof, "clocks": clk.summary(), "gpu_launches": rot["launches_per_step"] * steps,
            "would_fallback": rot["would_fallback"], "cache_generation_s": gen_s,
            "data": f"device-generated clustered unit rows (f4, {max(512, n_entries // 200)} clusters), host queries"}


def roofline(st, n_entries, dim, B, step_ms, rot, prof, n_rot, pk, cfg=None):
    """The dominant kernel's roofline entry (bench contract ④), from the library's launch counters."""
    dp = (dim + 63) // 64 * 64
    p8 = (dp + 127) // 128 * 128
    tensor = st["gemm_launches"] > 0  # which scan ran, from the library's own launch counters
    if not tensor and dp <= 1024:  # K2s: TMA-streamed int8 ring + per-row (scale, L1) + float64 queries + quantisation
        scan_bytes = n_entries * (p8 + 8) + B * (dp * 9 + 40)
        kname = "k_stream8_scan"
    elif not tensor:  # K2: fp16 ring
        scan_bytes = n_entries * dp * 2 + B * dp * 8
        kname = "k_gemv_scan"
    else:  # K3: fp16 ring + fp16 queries
        scan_bytes = n_entries * dp * 2 + B * dp * 2
        kname = "k_tc_scan_pair"
    fp16_bytes = n_entries * dim * 2 + B * dim * 2  # SURVEY.md §8(d)'s definition: an fp16 scan of the window
    flops = 2.0 * B * n_entries * dp
    hbm, tc_burst, tc_sust, src = pk
    # the dominant kernel's average duration: the rotation's mean step (one fused launch per step on the
    # small-batch path); on the tensor-core path the scan's share of the per-step cross-check (prep + pair),
    # split by the committed ncu launch list's per-kernel shares
    share = 1.0
    if rot["launches_per_step"] == 1:
        scan_s = step_ms * 1e-3
        timing = (f"CUDA events around the back-to-back timed steps on the library stream (rotation over {n_rot} "
                  "caches > L2), mean per launch")
    else:
        share = launch_share("k_tc_scan_pair", ("k_tc_prep", "k_tc_scan_pair"))
        scan_s = prof["scan_ms"] * 1e-3 * share
        timing = ("CUDA events around k_tc_prep + k_tc_scan_pair on the library stream (L2 flushed before each "
                  f"step), times the pair kernel's share {share:.3f} of that span in the committed ncu launch list")
    t_hbm = scan_bytes / (hbm * 1e9)
    t_tc = flops / (tc_burst * 1e12)
    bound = "hbm" if (not tensor or t_hbm >= t_tc) else "tensor"
    if bound == "hbm":
        roof = {"bound": "hbm", "achieved": scan_bytes / scan_s / 1e9, "peak": hbm, "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": flops / scan_s / 1e12, "peak": tc_burst, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    if roof["bound"] == "tensor":  # the back-to-back (power-limited) cuBLAS figure, beside the burst one
        roof["frac_of_sustained"] = roof["achieved"] / tc_sust
        roof["sustained_peak"] = tc_sust
    roof["peak_source"] = f"{src} (MEASURED_PEAKS.json)" if src == "measured" else "fallback (B200_PROFILING.md)"
    if roof["bound"] == "hbm":  # the measured peak is a read+write copy; a read-only scan can pass it
        roof["frac_of_spec"] = roof["achieved"] / 7700.0
        roof["spec_note"] = "7.7 TB/s: HGX B200 HBM3e nominal (B200_PROFILING.md)"
    roof["kernel"] = kname
    roof["algorithmic_bytes_per_launch"] = scan_bytes
    roof["bytes_definition"] = ("bytes the kernel must read: int8 ring rows + per-row (scale, L1) + queries"
                                if kname == "k_stream8_scan" else "fp16 ring rows + queries")
    roof["fp16_definition"] = {"bytes": fp16_bytes, "frac": fp16_bytes / scan_s / 1e9 / hbm,
                               "note": "SURVEY.md §8(d): N*D*2 + B*D*2 (an fp16 scan); the int8 copy reads half"}
    roof["flops_per_launch"] = flops
    roof["max_of_floors_frac"] = max(t_hbm, t_tc) / scan_s
    roof["step_roofline_frac"] = max(t_hbm, t_tc) / (step_ms * 1e-3)
    # ncu --set full captures exist for the C2 streamed scan and the C3 pair kernel only: their DRAM
    # bytes describe those shapes, so other sizes report no traffic rather than a borrowed figure
    captured = {"k_stream8_scan": "c2", "k_tc_scan_pair": "c3"}.get(kname)
    if cfg is not None and cfg == captured:
        roof["traffic"] = traffic_from_profiles(kname)
        roof["traffic_source"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch, profiles/ncu_summary.json"
    else:
        roof["traffic"] = None
        roof["traffic_source"] = f"no ncu --set full capture at this shape (captures: {kname} at {captured or 'none'})"
    roof["timing"] = timing
    return roof


class Dist:
    """torch.distributed plumbing for N > 1 (one process per GPU, NCCL): barrier and max over ranks."""

    def __init__(self):
        import torch
        import torch.distributed as td

        self.torch, self.td = torch, td
        self.rank = int(os.environ["RANK"])
        self.world = int(os.environ["WORLD_SIZE"])
        self.local = int(os.environ.get("LOCAL_RANK", self.rank))
        torch.cuda.set_device(self.local)
        td.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        self.torch.cuda.synchronize()
        self.td.barrier()

    def max_over_ranks(self, x: float) -> float:
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device="cuda")
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())


def run_sharded_c4(dist, n_total, B, steps, warmup, device=0):
    """C4: ONE cache of `n_total` entries sharded over the job's GPUs, one shard per rank (entries
    dealt round-robin by append position); at N = 1 the same code with one shard
    and no collective.  A step = B lookups: every rank's certified local scan
    (mc_retrieve_local_submit: no exhaustive-rescan launches behind it) -> NCCL all-gather of the
    B x 32-byte records -> merge and decisions on every rank (mc_merge_records_submit, decisions
    written to mapped host memory), read by mc_merge_records_wait one step later: two lookups in
    flight.  A merged MC_FLAG_NEED_RESCAN (a failed certificate on some shard) runs the second
    round (mc_rescan_local, all-gather, merge) on every rank.  Strong scaling: the cache and the
    batch stay fixed as N grows.  Timed by CUDA events on the step stream around the K steps
    (the host's enqueue and read-back of every step inside), max over ranks.  Caches are
    generated on the device (f4)."""
    import torch

    from paper_2503_11972_b200 import ThresholdTable, _native
    from paper_2503_11972_b200.workload import GeneratedWorkload

    G = dist.world if dist else 1
    g = dist.rank if dist else 0
    dim = 768
    wl = GeneratedWorkload(dim, n_clusters=max(512, n_total // 200), seed=17)
    n_local = (n_total - g + G - 1) // G  # positions p < n_total with p % G == g
    ring = _native.DeviceRing(-(-n_total // G), dim, device)
    ring.configure_shard(G, g)
    wl.fill(ring, n_local, row0=g * n_local)
    table = ThresholdTable.default()
    ring.set_table(table.pairs, table.total_steps)
    # the same trace on every rank: temporal locality (a drifting window of active clusters)
    Q = np.ascontiguousarray(wl.trace_queries((warmup + steps) * B).reshape(warmup + steps, B, dim))
    # batch 1: every request also stores its generated image (FIFO insert, evicting the oldest
    # entry of the full cache); global position n_total + i lands on shard (n_total + i) % G only
    inserts = B == 1
    new_rows = wl.images(Q[:, 0]) if inserts else None
    n_ins = 0  # inserts so far = the oldest live global position (the cache is full)
    if B > 4:  # batches DMA'd straight from the page-locked query array (no staging copy)
        _native.register_host(Q)
    nb = B * 32
    dev = torch.device("cuda", device)
    cs = torch.cuda.Stream(dev)
    NS = _native.DeviceRing.MERGE_SLOTS  # lookups in flight: step i+1 is enqueued before step i is read
    local = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(NS)]
    gathered = [torch.empty(G * nb, dtype=torch.uint8, device=dev) for _ in range(NS)]
    hits = rescans = 0
    # A batch enters the job once: each rank uploads its 1/G of the rows, and the ranks
    # all-gather the batch over NVLink (instead of G host uploads of the whole batch).
    split = dist is not None and B > 4 and B % G == 0 and (G > 1 or os.environ.get("MC_C4_SPLIT_UPLOAD"))
    if split:
        Qt = torch.from_numpy(Q)  # page-locked above: the slice copies are DMAs
        part = B // G
        local_q = [torch.empty(part * dim, dtype=torch.float64, device=dev) for _ in range(NS)]
        full_q = [torch.empty(B * dim, dtype=torch.float64, device=dev) for _ in range(NS)]

    csp = cs.cuda_stream
    gptr = [t.data_ptr() for t in gathered]  # raw pointers: no per-step tensor attribute lookups

    p0s = [0] * NS  # oldest live global position at each in-flight lookup's submit

    def submit(i):
        nonlocal n_ins
        j = i % NS
        p0 = p0s[j] = n_ins
        if G == 1 and not split:  # no collective: the ring's own calls order themselves after csp
            ring.retrieve_local_submit(Q[i], gptr[j], csp)
            ring.merge_submit(gptr[j], G, B, p0, csp, j)
        else:
            submit_collective(i, j, p0)
        if inserts:  # this request's image, appended after its lookup was enqueued
            if (n_total + n_ins) % G == g:
                ring.append1(new_rows[i])
            n_ins += 1

    def submit_collective(i, j, p0):
        with torch.cuda.stream(cs):
            if split:
                local_q[j].copy_(Qt[i, g * part:(g + 1) * part].reshape(-1), non_blocking=True)
                dist.td.all_gather_into_tensor(full_q[j], local_q[j])
                ring.retrieve_local_device(full_q[j], B, local[j], cs.cuda_stream)
                dist.td.all_gather_into_tensor(gathered[j], local[j])
            elif G > 1:  # the scan without the exhaustive rescan behind it (second round on demand)
                ring.retrieve_local_submit(Q[i], local[j], cs.cuda_stream)
                dist.td.all_gather_into_tensor(gathered[j], local[j])
            else:
                ring.retrieve_local_submit(Q[i], gathered[j], cs.cuda_stream)
        ring.merge_submit(gathered[j], G, B, p0, cs.cuda_stream, j)

    def collect(i):
        nonlocal hits, rescans
        j = i % NS
        live, sim, k, flags = ring.merge_wait(j)
        if not split and (flags & _native.MC_FLAG_NEED_RESCAN).any():  # same decision on every rank
            rescans += 1
            with torch.cuda.stream(cs):
                own = local[j] if G > 1 else gathered[j]
                ring.rescan_local(Q[i], own, cs.cuda_stream)
                if G > 1:
                    dist.td.all_gather_into_tensor(gathered[j], local[j])
            ring.merge_submit(gathered[j], G, B, p0s[j], cs.cuda_stream, j)
            live, sim, k, flags = ring.merge_wait(j)
        hits += int((flags & _native.MC_FLAG_HIT).astype(bool).sum())

    def run(first, last):  # NS - 1 lookups stay in flight while the host prepares the next
        for i in range(first, last):
            submit(i)
            if i - first >= NS - 1:
                collect(i - NS + 1)
        for i in range(max(first, last - NS + 1), last):
            collect(i)

    run(0, warmup)
    hits = rescans = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    run(warmup, warmup + steps)
    e1.record(cs)
    e1.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    if dist:
        dt = dist.max_over_ranks(dt)
    if B > 4:
        _native.unregister_host(Q)
    ring.close()
    return {"workload": f"C4: one {n_total:,}-entry cache x {dim} sharded over {G} GPU(s) (round-robin by append "
                        f"position), batch {B}, local scan + NCCL all-gather of {B}x32-byte records + merge",
            "value": B * steps / dt, "unit": "lookups/s", "ms_per_step": 1e3 * dt / steps, "batch": B,
            "n_gpus": G, "rows_per_gpu": n_local, "scaling": "strong", "hit_fraction": hits / (B * steps),
            "query_upload": ("1/G of the batch per rank + NCCL all-gather of the queries" if split
                             else "the whole batch from the host on every rank"),
            "second_rounds": rescans,
            "trace": ("temporal locality: each request's cluster drawn from a window of 64 active clusters that "
                      "advances one cluster every 256 requests (workload.py:93-121's lifetimes, vectorised)"
                      + ("; every request also inserts its generated image (FIFO, evicting the oldest of the full "
                         "cache) on the owning shard" if inserts else "")),
            "pipelining": f"{NS} lookups in flight (step i+1 enqueued before step i's decisions are read)",
            "timing": "CUDA events on the step stream around the timed steps (the host's enqueue and read-back "
                      "of every step inside; the last step's decisions read before the end event is waited on), "
                      "max over ranks"}


def launch_share(kernel: str, group) -> float:
    """kernel's share of the summed durations of `group` in the committed ncu launch list."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())["launch_list_mean_us"]
        tot = sum(d[k] for k in group)
        return d[kernel] / tot if tot > 0 else 1.0
    except Exception:
        return 1.0


def traffic_from_profiles(kernel: str):
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def _reference_cache_module():
    """The UNMODIFIED reference package staged under baseline/_ref (scripts/stage_reference.sh), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mixserve" / "cache.py").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import mixserve.cache as mc

        return mc
    except Exception:
        return None


def reference_arm(args):
    """The reference's own CPU path on the box's host cores, same workload as our arm's headline.

    Each step = a bounded sample of the C2 workload: `per_step` sequential
    SemanticCache.retrieve + add calls (the reference has no batch API) against
    the 100k x 768 cache.  Runs the real `mixserve.cache.SemanticCache` when the
    reference is staged under baseline/_ref (kind "reference"); otherwise the
    oracle port of the same algorithm (kind "port").
    """
    per_step = 4
    total = args.warmup + args.steps
    rows, Q, new_rows = make_workload(768, 100_000, total * per_step + 8)
    n, dim = rows.shape
    mc = _reference_cache_module()
    if mc is not None:
        cache = mc.SemanticCache(capacity=n, dim=dim)
        for i, v in enumerate(rows):
            cache.insert(mc.CacheEntry(f"e{i}", v, "large", i, 0.0))
        table = mc.ThresholdTable.default()
        kind, what = "reference", f"mixserve.cache.SemanticCache from baseline/_ref (unmodified reference)"
        lookup = lambda q: cache.retrieve(q, table)  # noqa: E731
        insert = lambda j: cache.add(f"n{j}", new_rows[j], "large", 1.0 + j)  # noqa: E731
    else:
        from oracle.retrieval import OracleCache, OracleEntry, OracleTable

        o = OracleCache(n, dim)
        for i, v in enumerate(rows):
            o.insert(OracleEntry(f"e{i}", v, "large", i, 0.0))
        t = OracleTable()
        kind, what = "port", "oracle/retrieval.py (float64 numpy port of cache.py:244-260)"
        lookup = lambda q: o.retrieve(q, t)  # noqa: E731
        insert = lambda j: o.insert(OracleEntry(f"n{j}", new_rows[j], "large", n + j, 0.0))  # noqa: E731
    from oracle.retrieval import blas_info

    j = 0
    times = []
    for _ in range(total):
        t0 = time.perf_counter()
        for _ in range(per_step):
            lookup(Q[j])
            insert(j)
            j += 1
        times.append(time.perf_counter() - t0)
    timed = sum(times[args.warmup:])
    value = args.steps * per_step / timed
    threads = blas_threads()
    cb = {"value": value, "unit": "lookups/s", "cores": threads or os.cpu_count(), "kind": kind,
          "blas_threads": threads, "host_cpu_count": os.cpu_count(),
          "sample": f"{args.steps} steps x {per_step} sequential retrieve+add calls on a {n}x{dim} float64 cache; "
                    f"{what}; {blas_info()}"}
    return {
        "metric": METRIC, "value": value, "unit": "lookups/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * timed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA, "config": dict(C2_CONFIG),
        "impl": "reference", "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-big", action="store_true", help="skip the 1M / 10M-entry single-GPU lines")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.warmup < 3:
        args.warmup = 3

    if args.impl == "reference":
        if rank != 0:
            return  # rank 0 alone runs the CPU reference arm
        print(json.dumps(reference_arm(args)))
        return

    dist = Dist() if (world > 1 or os.environ.get("BENCH_DIST")) else None  # BENCH_DIST: exercise N=1 under torchrun
    device = dist.local if dist else 0
    pk = peaks()
    flush = 256 << 20
    c2 = run_config("c2", 768, 100_000, 1, args.steps, args.warmup, True, flush, pk, device=device, dist=dist,
                    e2e_steps=3000)
    line = {
        "metric": METRIC,
        "value": c2["value"], "unit": "lookups/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": c2["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int8 scan (exact int32 dot, certified per-row bounds) / f64 rescoring",
        "data": DATA,
        "config": dict(C2_CONFIG, l2="inputs larger than L2: steps rotate over 4 caches of this shape (4 x 77.6 MB "
                                     "int8 scan copies), timed back to back",
                       parallelism=f"replicas{world}" if world > 1 else "single"),
        "e2e": c2["e2e"], "roofline": c2["roofline"], "clocks": c2["clocks"], "gpu_launches": c2["gpu_launches"],
        "profile": c2["profile"], "native_stats": c2["stats"],
    }
    if not args.no_c3:
        c3 = run_config("c3", 1024, 100_000, 256, min(60, max(20, args.steps // 10)), args.warmup, False, flush, pk,
                        device=device, n_rot=2, dist=dist, e2e_steps=100)
        line["c3"] = {"workload": "C3: 100k entries, 1024-dim, batch-256 lookups", "value": c3["value"],
                      "unit": "lookups/s", "ms_per_step": c3["ms_per_step"], "e2e": c3["e2e"],
                      "roofline": c3["roofline"], "clocks": c3["clocks"], "gpu_launches": c3["gpu_launches"],
                      "profile": c3["profile"]}
    if not args.no_c3:  # C1: the reference's default size, L2-resident by design -> reported as latency
        c1 = run_config("c1", 768, 10_000, 1, max(200, args.steps), args.warmup, True, 0, pk, device=device, n_rot=1,
                        dist=dist, e2e_steps=2000)
        line["c1"] = {"workload": "C1: 10k-entry FIFO cache (reference default), 768-dim, batch-1 lookup + insert",
                      "device_latency_us": 1e3 * c1["profile"]["step_ms"],
                      "device_latency_timing": "CUDA events around each isolated lookup (event pair and launch "
                                               "latency included, no overlap with a neighbour)",
                      "back_to_back_us": 1e3 * c1["ms_per_step"], "value": c1["value"], "unit": "lookups/s",
                      "e2e": c1["e2e"], "roofline": c1["roofline"], "clocks": c1["clocks"],
                      "l2": "resident (15.4 MB int8 copy): latency, not HBM, is the figure of merit"}
    if not args.no_big and not dist:  # C4 / C5 shapes on one GPU (device-generated caches, f4)
        big = {}
        for key, n, B, k in (("c4_b1", 1_000_000, 1, max(args.steps, 50)), ("c4_b256", 1_000_000, 256, 20),
                             ("c5_b1", 10_000_000, 1, 20), ("c5_b256", 10_000_000, 256, 6)):
            label = (f"{'C4' if n == 1_000_000 else 'C5'} shape on ONE GPU: {n:,} entries x 768, batch {B}"
                     + ("" if n == 1_000_000 else " (all 10M entries in this GPU's HBM: 61.4 GB float64 + 15.4 GB fp16"
                                                   " + 7.7 GB int8)"))
            try:
                big[key] = run_generated(label, None, 768, n, B, k, args.warmup, flush, pk, device=device)
            except Exception as exc:  # reported, never fatal to the headline line
                big[key] = {"workload": label, "error": f"{type(exc).__name__}: {exc}"}
        line["single_gpu_large"] = big
    if not args.no_big:  # the path's exchange step: one 1M-entry cache sharded over the job's GPUs
        line["c4_sharded"] = {}
        for B, k in ((1, max(args.steps, 50)), (256, 20)):
            try:
                line["c4_sharded"][f"b{B}"] = run_sharded_c4(dist, 1_000_000, B, k, args.warmup, device=device)
            except Exception as exc:  # reported, never fatal to the headline line
                line["c4_sharded"][f"b{B}"] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0:
        line["cpu_baseline"] = cpu_baseline(c2["rows"], c2["Q"], c2["new_rows"], insert=True, seconds=args.cpu_seconds)
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.td.destroy_process_group()


if __name__ == "__main__":
    main()
