#!/usr/bin/env python
"""Benchmark: layout conversion + transfer of record collections on B200.

Workload (BASELINE.json configs[4], the north-star shape): a collection of
1,000,000,000 Obj8 records (8 x f32/i32 fields, 32-byte packed AoS) sharded by
contiguous object-index range over the N GPUs of one box. One step converts
every rank's AoS shard into per-field planes (SoA) in HBM through the public
API (copy_collection -> b200-convert -> one launch of the conversion engine).
No collective on the data path (objects are independent), so `scaling` is
"strong": the 1B-object total is fixed as N grows.

value      whole-job algorithmic GB/s (64 B per object: 32 read + 32 written),
           inputs resident in HBM, device time (CUDA events), max over ranks
e2e        the same metric through copy_collection with the AoS in pinned HOST
           memory: chunked H2D | convert | result read-back inside the timed
           region (bounded sample per rank, stated in e2e.sample)
roofline   the conversion kernel vs the measured HBM copy peak
cpu_baseline  the reference's per-leaf numpy path (oracle port), 1 core, on a
           bounded sample (rank 0, N=1 only)

--impl reference runs the reference's CPU path (oracle port) sharded over all
host cores instead, on rank 0 only.
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "layout-convert+transfer GB/s and objects/s vs HBM roofline, 1/2/4/8 B200"
UNIT = "GB/s"
WORKLOAD = "config5: Obj8 AoS->SoA (8 x f32/i32, 32 B records), 1e9 objects sharded by object index"
BYTES_PER_OBJECT = 64


def _peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int) -> None:
        self.device = device
        self.lines: list[str] = []
        self.proc = None
        self.thread = None

    def start(self) -> None:
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self) -> None:
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _cpu_info() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- our arm -------------------------------------------------------------------------------------

def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = _dist()
    # SK_BENCH_DEVICE / SK_BENCH_BACKEND exist only to exercise the multi-rank
    # code path on a single GPU (all ranks on one device, gloo plumbing).
    local = int(os.environ.get("SK_BENCH_DEVICE", local))
    backend = os.environ.get("SK_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    tdev = f"cuda:{local}" if backend == "nccl" else "cpu"

    import paper_2511_04853_b200 as sk
    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import layouts as ly, memctx as mc, schema as sc, shard, transfer as tr
    from paper_2511_04853_b200 import workloads as wl

    dev = local
    cuda = mc.ContextInfo.cuda(dev)

    def barrier():
        nat.sync(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def min_over_ranks(x: float) -> float:
        return -max_over_ranks(-x)

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def device_collection(schema, kind, n, ipc=False):
        c = sk.Collection(schema, kind, mc.ContextInfo.cuda(dev, ipc=True) if ipc else cuda)
        with mc.execution_scope(mc.CUDA):
            c.reserve(n)
        with c.layout.engine_ops():
            c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
        return c

    n_total = args.objects
    free_b, _ = torch.cuda.mem_get_info(dev)
    lo, hi = shard.shard_range(n_total, rank, world)
    n = hi - lo
    need = (3 if world > 1 else 2) * n * 32 * (world if os.environ.get("SK_BENCH_DEVICE") else 1)
    if need > free_b * 0.9:
        raise SystemExit(f"rank {rank}: shard of {n} objects needs {need / 1e9:.1f} GB, {free_b / 1e9:.1f} GB free")

    aos = device_collection(wl.OBJ8_SCHEMA, ly.AOS, n, ipc=world > 1)  # exportable: the P2P leg pulls it
    soa = device_collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, n)
    # the global 1e9-record image is splitmix64(seed, word); this shard is its slice
    wl.fill_random_device(aos.layout._struct_buf.ptr, n * 32, seed=SEED, device=dev, first_word=lo * 4)

    def step():
        tr.copy_collection(soa, aos, {"async": True})

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks(dev) if rank == 0 else None
    if clocks:
        clocks.start()
    evs = [nat.Event() for _ in range(args.steps + 1)]
    barrier()
    evs[0].record(dev)
    for k in range(args.steps):
        step()
        evs[k + 1].record(dev)
    barrier()
    clk = clocks.stop() if clocks else None
    per_launch = [evs[k].elapsed_ms(evs[k + 1]) for k in range(args.steps)]
    local_ms = evs[0].elapsed_ms(evs[-1]) / args.steps
    ms = max_over_ranks(local_ms)
    value = n_total * BYTES_PER_OBJECT / (ms / 1e3) / 1e9
    mine = n * BYTES_PER_OBJECT / (statistics.mean(per_launch) / 1e3) / 1e9  # this rank's HBM GB/s
    launch_ms = max_over_ranks(statistics.mean(per_launch))
    achieved = n * BYTES_PER_OBJECT / (launch_ms / 1e3) / 1e9  # per GPU, slowest rank's launch time
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)

    # parity of the timed output at full scale (the run fails on any mismatch)
    parity = verify_obj8_shard(aos, soa, n, lo, dev, rank)

    # ---- e2e: pinned HOST AoS -> device SoA through the public API, result read back ----
    m = min(args.e2e_objects, n)
    host = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
    host.resize(m)
    nat.memcpy(host.layout._struct_buf.ptr, aos.layout._struct_buf.ptr, m * 32, dev)  # same records as the shard head
    dst = device_collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, m)
    result = np.empty(8, np.uint32)
    tails = [dst.layout.plane_address(dst.plan.leaf(f"f{i}")) + (m - 1) * 4 for i in range(8)]

    def e2e_step():
        tr.copy_collection(dst, host)  # H2D + convert, pipelined; returns when done
        for i, p in enumerate(tails):  # device->host read of the step's result (last record)
            nat.memcpy(result.ctypes.data + 4 * i, p, 4, dev)
        nat.sync(dev)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    e0, e1 = nat.Event(), nat.Event()
    e2e_steps = max(2, min(args.steps, 5))
    barrier()
    e0.record(dev)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(dev)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_ms(e1) / e2e_steps)
    m_total = sum_over_ranks(m)
    e2e_value = m_total * BYTES_PER_OBJECT / (e2e_ms / 1e3) / 1e9
    # the link the e2e leg is bound by: pinned host -> HBM copy of the same bytes
    l0, l1 = nat.Event(), nat.Event()
    nat.memcpy(aos.layout._struct_buf.ptr, host.layout._struct_buf.ptr, m * 32, dev)
    barrier()
    l0.record(dev)
    for _ in range(3):
        nat.memcpy(aos.layout._struct_buf.ptr, host.layout._struct_buf.ptr, m * 32, dev)
    l1.record(dev)
    barrier()
    h2d_gbs = min_over_ranks(m * 32 * 3 / (l0.elapsed_ms(l1) / 1e3) / 1e9)
    host.free()
    # the same through PAGEABLE host memory (the reference's default placement, ContextInfo.host()):
    # the pipeline stages it through pinned buffers; a smaller bounded sample
    mp_ = min(m, args.e2e_objects // 4)
    page = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.host())
    page.resize(mp_)
    nat.memcpy(page.layout._struct_buf.ptr, aos.layout._struct_buf.ptr, mp_ * 32, dev)
    nat.sync(dev)
    tails_p = [dst.layout.plane_address(dst.plan.leaf(f"f{i}")) + (mp_ - 1) * 4 for i in range(8)]

    def e2e_pageable():
        tr.copy_collection(dst, page)
        for i, p in enumerate(tails_p):
            nat.memcpy(result.ctypes.data + 4 * i, p, 4, dev)
        nat.sync(dev)

    f0, f1 = nat.Event(), nat.Event()
    f0.record(dev)
    e2e_pageable()  # the first transfer page-locks the buffer (memctx.pin_for_transfer)
    f1.record(dev)
    nat.sync(dev)
    first_ms = max_over_ranks(f0.elapsed_ms(f1))
    q0, q1 = nat.Event(), nat.Event()
    barrier()
    q0.record(dev)
    for _ in range(e2e_steps):
        e2e_pageable()
    q1.record(dev)
    barrier()
    pg_ms = max_over_ranks(q0.elapsed_ms(q1) / e2e_steps)
    pageable = {"value": round(sum_over_ranks(mp_) * BYTES_PER_OBJECT / (pg_ms / 1e3) / 1e9, 2), "unit": UNIT,
                "ms_per_step": round(pg_ms, 3), "h2d_bytes_per_step": mp_ * 32 * world,
                "first_call_ms": round(first_ms, 3),
                "sample": f"{mp_} objects per rank in pageable host memory (numpy, ContextInfo.host()) -> device "
                          "per_field via copy_collection, then D2H of the last converted record; the first "
                          "transfer page-locks the buffer once (first_call_ms includes it), the timed steps "
                          "reuse it"}
    page.free()
    dst.free()

    # ---- layout-changing peer pull (config 5b): rank r converts the AoS shard
    # owned by rank (r+1) % N into planes on its own GPU; the kernel reads the
    # peer's HBM over NVLink (CUDA IPC mapping), writes local HBM.
    p2p = None
    if world > 1 and not args.no_p2p:
        from paper_2511_04853_b200 import shard as sh

        # setup failures (no IPC/peer access on some box) are agreed on by every
        # rank so nobody is left waiting in a collective; the leg then reports why
        err = ""
        mine = remote = pulled = None
        try:
            mine = sh.export_collection(aos)
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            err = f"export: {e}"
        every = [None] * world
        dist.all_gather_object(every, mine)
        src_rank = (rank + 1) % world
        if not err:
            try:
                remote = sh.import_collection(wl.OBJ8_SCHEMA, every[src_rank], dev)
                pulled = device_collection(wl.OBJ8_SCHEMA, ly.PER_FIELD, remote.size())
            except Exception as e:  # noqa: BLE001
                err = f"import from rank {src_rank}: {e}"
        ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64, device=tdev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if ok.item() < 1.0:
            for c in (remote, pulled):
                if c is not None:
                    c.free()
            p2p = {"unavailable": "; ".join(f"rank {r}: {e}" for r, e in enumerate(errs) if e)[:400]}
    if world > 1 and not args.no_p2p and p2p is None:
        n_src = remote.size()

        def p2p_step():
            tr.copy_collection(pulled, remote, {"async": True})

        for _ in range(2):
            p2p_step()
        barrier()
        a, b = nat.Event(), nat.Event()
        a.record(dev)
        for _ in range(args.steps):
            p2p_step()
        b.record(dev)
        barrier()
        p_ms = max_over_ranks(a.elapsed_ms(b) / args.steps)
        p_total = sum_over_ranks(n_src)
        per_gpu_link = max_over_ranks(n_src) * 32 / (p_ms / 1e3) / 1e9
        # the link itself: a plain copy engine read of the same peer bytes into local HBM
        cp_bytes = min(n_src * 32, 1 << 30)
        tmp = nat.malloc(dev, cp_bytes)
        rptr = remote.layout._struct_buf.ptr
        nat.memcpy(tmp, rptr, cp_bytes, dev)
        barrier()
        c0, c1 = nat.Event(), nat.Event()
        c0.record(dev)
        for _ in range(5):
            nat.memcpy(tmp, rptr, cp_bytes, dev)
        c1.record(dev)
        barrier()
        peer_copy = min_over_ranks(cp_bytes * 5 / (c0.elapsed_ms(c1) / 1e3) / 1e9)
        nat.free(dev, tmp)
        p2p = {"value": round(p_total * BYTES_PER_OBJECT / (p_ms / 1e3) / 1e9, 2), "unit": UNIT,
               "ms_per_step": round(p_ms, 3), "objects_total": int(p_total),
               "nvlink_read_gbs_per_gpu": round(per_gpu_link, 1),
               "peer_copy_gbs_measured": round(peer_copy, 1), "frac_of_peer_copy": round(per_gpu_link / peer_copy, 3),
               "nvlink_nominal_gbs": 900.0, "frac_of_nominal": round(per_gpu_link / 900.0, 3),
               "note": "GPU r pulls rank (r+1)%N's AoS shard through a CUDA IPC mapping (32 B/object over "
                       "NVLink read, 32 B/object local HBM write); peer_copy = cudaMemcpyAsync of the same "
                       "peer bytes into local HBM, measured in this run (min over ranks)"}
        barrier()
        remote.free()
        pulled.free()
        barrier()

    extra = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_extra:
        extra = run_extras(args, dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import cpu_baseline

        cb = cpu_baseline.reference_single_core(args.cpu_objects, budget_s=args.cpu_seconds)
        if cb is not None:
            what = ("soakit's own copy_collection(per_field, aos) on host collections (per-leaf-default, "
                    "transfer.py:171-236) from baseline/_ref")
        else:
            cb = dict(cpu_baseline.single_core(args.cpu_objects, budget_s=args.cpu_seconds), kind="port")
            what = "reference per-leaf numpy path (transfer.py:196-228) restated in oracle/cpu_baseline.py"
        cpu = {"value": round(cb["gbs"], 3), "unit": UNIT, "cores": 1, "kind": cb["kind"],
               "objects_per_s": round(cb["objects_per_s"]),
               "sample": f"{args.cpu_objects} Obj8 objects, {what}, mean of the fastest samples "
                         f"(bench.py:214-215); host: {os.cpu_count()} x {_cpu_info()}"}
        if extra:
            # the reference's CPU path beside each extra config (one core, bounded samples)
            pc = cpu_baseline.per_config(budget_s=1.5)
            for key, val in (cpu_baseline.reference_per_config(budget_s=1.5) or {}).items():
                pc[key] = val  # configs 1-3 through soakit itself when baseline/_ref is present
            if "config2_reconstruct" in pc and "config2_reconstruct_64_events" in extra:
                r = pc["config2_reconstruct"]
                extra["config2_reconstruct_64_events"]["cpu_reference_1core"] = {
                    k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}
                extra["config2_reconstruct_64_events"]["gpu_over_cpu_1core"] = round(
                    extra["config2_reconstruct_64_events"]["events_per_s"] / r["events_per_s"], 1)
            pairs = {"config1_obj8_1M": ("config1_obj8", "device_gbs"),
                     "config2_sensor_64x190096": ("config2_sensor", "device_gbs"),
                     "config3_jagged_1M": ("config3_jagged", "gbs"),
                     "config4_aosoa_100M": ("config4_aosoa", "gbs")}
            for key, (ck, gkey) in pairs.items():
                if key in extra and ck in pc:
                    c = pc[ck]
                    label = "cpu_reference_1core" if c.get("kind") == "reference" else "cpu_port_1core"
                    extra[key][label] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in c.items()}
                    extra[key]["gpu_over_cpu_1core"] = round(extra[key][gkey] / c["gbs"], 1)
            if "config3_jagged_1M" in extra and pc.get("config3_jagged", {}).get("kind") == "reference":
                jf = extra["config3_jagged_1M"]["jagged_fill"]  # the same call on both sides
                jf["over_reference_jagged_fill_1core"] = round(
                    jf["members_per_s"] / pc["config3_jagged"]["members_per_s"], 1)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = _traffic(n)
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": f"synthetic (splitmix64 record images generated on-device, seed {SEED})",
        "config": {"workload": WORKLOAD, "objects_total": n_total, "objects_per_gpu": n, "record_bytes": 32,
                   "algorithmic_bytes_per_object": BYTES_PER_OBJECT,
                   "sharding": "contiguous object-index ranges, no data-path collective",
                   "l2": "inputs (32 GB AoS at N=1) far larger than the 126 MB L2; no flush needed",
                   "timing": "CUDA events on the library stream, barrier + sync both sides, max over ranks"},
        "objects_per_s": round(n_total / (ms / 1e3)),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "sk::conv::convert_kernel_t<GenericTransform> (word-mode AoS->planes, TMA bulk "
                               "in/out); traffic from profiles/r02_obj8_a2p.ncu-rep scaled to this launch",
                     "per_rank_frac": [round(x / peak, 4) for x in per_rank],
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (torch copy, read+write)" if peaks else
                                    "fallback 6650 GB/s (B200_PROFILING.md)"},
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": m * 32 * world,
                "d2h_bytes_per_step": 32 * world, "ms_per_step": round(e2e_ms, 3),
                "h2d_link_gbs_measured": round(h2d_gbs, 1),
                "frac_of_h2d_link": round(m * 32 * world / (e2e_ms / 1e3) / 1e9 / (h2d_gbs * world), 3),
                "sample": f"{m} objects per rank in pinned host memory -> device per_field via copy_collection "
                          "(chunked H2D | convert | on 3 streams), then D2H of the last converted record",
                "result_readback": "32 B per rank per step (the last converted record, 8 planes x 4 B) of the "
                                   f"{m * 32} B converted: the converted planes stay in HBM, where the "
                                   "application's next kernel reads them",
                "pageable_host": pageable},
        "gpu_launches": args.steps,
        "clocks": clk,
        "cpu_baseline": cpu,
        "parity": parity,
    }
    if p2p:
        line["p2p"] = p2p
    if extra:
        line["configs"] = extra
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


SEED = 20251104


def verify_obj8_shard(aos, soa, n: int, lo: int, dev: int, rank: int) -> dict:
    """Check the converted shard two ways; SystemExit on any mismatch.

    1. Sampled records against the CPU oracle (oracle/restate.splitmix_image:
       the input image restated from its definition, not read back): the
       first and last 4096-record tiles, the tiles that start at AoS byte
       offsets 2^32, 2^33, 2^34 (past any 32-bit offset), and 64 seeded
       random tiles. Semantics: transfer.py:196-233 / layouts.py:573-598.
    2. Every record: the planes are converted back to AoS (K2) into a third
       buffer and compared byte-for-byte with the input AoS on the device
       (sk_compare_bytes), so the whole 32 GB image is covered."""
    import ctypes as C

    import numpy as np

    from oracle import restate
    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import layouts as ly, memctx as mc, schema as sc, transfer as tr
    from paper_2511_04853_b200 import workloads as wl
    import paper_2511_04853_b200 as sk

    t = min(4096, n)
    starts = {0, n - t}
    for e in (32, 33, 34):
        r = (1 << e) // 32
        if r + t <= n:
            starts.add(r)
    rng = np.random.default_rng(1234 + rank)
    starts.update(int(x) for x in rng.integers(0, max(1, n - t + 1), 64))
    got = np.empty(t * 4, np.uint8)
    for r0 in sorted(starts):
        want = restate.splitmix_image(SEED, lo * 4, r0 * 32, t * 32).view(wl.OBJ8_AOS_DTYPE)
        for i in range(8):
            nat.memcpy(got.ctypes.data, soa.layout.plane_address(soa.plan.leaf(f"f{i}")) + r0 * 4, got.nbytes, dev)
            nat.sync(dev)
            if got.tobytes() != np.ascontiguousarray(want[f"f{i}"]).tobytes():
                raise SystemExit(f"rank {rank}: plane f{i} of records [{r0}, {r0 + t}) differs from the oracle")
    back = sk.Collection(wl.OBJ8_SCHEMA, ly.AOS, mc.ContextInfo.cuda(dev))
    with mc.execution_scope(mc.CUDA):
        back.reserve(n)
    tr.copy_collection(back, soa)
    bad = nat.malloc(dev, 8)
    nat.call("sk_compare_bytes", back.layout._struct_buf.ptr, aos.layout._struct_buf.ptr, n * 32, bad,
             nat.stream(dev))
    cnt = C.c_uint64(0)
    nat.memcpy(C.addressof(cnt), bad, 8, dev)
    nat.sync(dev)
    nat.free(dev, bad)
    back.free()
    if cnt.value:
        raise SystemExit(f"rank {rank}: AoS -> planes -> AoS round trip differs in {cnt.value} bytes")
    return {"sampled_vs_oracle": f"{len(starts)} tiles of {t} records (first, last, AoS byte offsets 2^32/2^33/2^34, "
                                 "64 random) x 8 planes, byte-exact vs oracle/restate.splitmix_image",
            "full_round_trip": f"{n} records: planes -> AoS (K2) == input AoS, 0 of {n * 32} bytes differ "
                               "(sk_compare_bytes on the device)"}


def config2_api_paths(a2, p2, h2, noise, cells, dev, peak, queued, timed) -> dict:
    """Config 2 through the reference-facing API rather than the fused extension:
    copy_collection + funcs.calibrate_energy() + funcs.get_noise() (the
    reference's prepare phase, bench.py:174-178), batched and per event with the
    reference's protocol (mean of the 10 fastest of 50 reps cycling 10 events,
    bench.py:214-289), plus the K5 kernels alone against their roofline."""
    import time

    import numpy as np

    import paper_2511_04853_b200 as sk
    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import layouts as ly, memctx as mc, schema as sc, sensor, transfer as tr
    from paper_2511_04853_b200.devarray import DeviceArray

    def api_batch():  # pinned AoS -> device planes, then the two behaviors (separate K5 kernels)
        tr.copy_collection(p2, h2)
        with mc.execution_scope(mc.CUDA):
            p2.funcs.calibrate_energy()
            p2.funcs.get_noise().free()

    ms_api = timed(api_batch, steps=3, warmup=1)

    def api_fused():  # the same reference-API sequence with the fusion option: one HBM pass
        tr.copy_collection(p2, h2, {"fuse": "sensor_funcs"})
        with mc.execution_scope(mc.CUDA):
            p2.funcs.calibrate_energy()
            p2.funcs.get_noise()

    ms_api_fused = timed(api_fused, steps=3, warmup=1)
    ms_api_fused_dev = queued(lambda: tr.copy_collection(p2, a2, {"async": True, "fuse": "sensor_funcs"}), steps=10)

    def api_device():  # the same three steps on device-resident AoS records
        tr.copy_collection(p2, a2, {"async": True})
        sensor.calibrate_collection(p2, sync=False)
        sensor.noise_for_collection(p2, noise, sync=False)

    ms_api_dev = queued(api_device, steps=10)
    ms_cal = queued(lambda: sensor.calibrate_collection(p2, sync=False), steps=20)
    ms_noise = queued(lambda: sensor.noise_for_collection(p2, noise, sync=False), steps=20)

    # per event, the reference's protocol
    ev = 436 * 436
    pinned = mc.ContextInfo.pinned()
    events = []
    for e in range(10):
        c = sk.Collection(sensor.SENSOR_SCHEMA, ly.AOS, pinned)
        c.resize(ev)
        nat.memcpy(c.layout._struct_buf.ptr, a2.layout._struct_buf.ptr + e * ev * 30, ev * 30, dev)
        events.append(c)
    nat.sync(dev)
    d1 = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, mc.ContextInfo.cuda(dev))
    n1 = DeviceArray(ev, np.float32, mc.ContextInfo.cuda(dev))

    def protocol(rep) -> float:
        rep(0)
        samples = []
        for r in range(50):
            t0 = time.perf_counter()
            rep(r % 10)
            samples.append(time.perf_counter() - t0)
        return sum(sorted(samples)[:10]) / 10 * 1e3

    def api_event(e):
        tr.copy_collection(d1, events[e])
        sensor.calibrate_collection(d1)
        sensor.noise_for_collection(d1, n1)

    ms_ev_api = protocol(api_event)

    def api_fused_event(e):
        tr.copy_collection(d1, events[e], {"fuse": "sensor_funcs"})
        with mc.execution_scope(mc.CUDA):
            d1.funcs.calibrate_energy()
            d1.funcs.get_noise()

    ms_ev_api_fused = protocol(api_fused_event)
    ms_ev_fused = protocol(lambda e: sensor.transfer_calibrate(d1, events[e], n1))
    for c in events:
        c.free()
    d1.free()
    n1.free()
    return {
        "api_pinned_e2e_ms": round(ms_api, 3),
        "api_pinned_e2e_cells_per_s": round(cells / ms_api * 1e3),
        "api_device_ms": round(ms_api_dev, 3),
        "api_device_gbs": round(cells * 64 / ms_api_dev / 1e6, 1),
        "api_fused_option_pinned_e2e_ms": round(ms_api_fused, 3),
        "api_fused_option_device_ms": round(ms_api_fused_dev, 3),
        "api_fused_option_device_gbs": round(cells * 64 / ms_api_fused_dev / 1e6, 1),
        "k5_calibrate": {"ms": round(ms_cal, 4), "gbs": round(cells * 20 / ms_cal / 1e6, 1),
                         "frac": round(cells * 20 / ms_cal / 1e6 / peak, 3),
                         "bytes_per_cell": "20 (counts 8 + A 4 + B 4 read, energy 4 written)",
                         "roofline": _cfg_roofline("config2_k5_calibrate", cells * 20, ms_cal, cells, peak)},
        "k5_noise": {"ms": round(ms_noise, 4), "gbs": round(cells * 17 / ms_noise / 1e6, 1),
                     "frac": round(cells * 17 / ms_noise / 1e6 / peak, 3),
                     "bytes_per_cell": "17 (energy 4 + nA 4 + nB 4 + noisy 1 read, noise 4 written)",
                     "roofline": _cfg_roofline("config2_k5_noise", cells * 17, ms_noise, cells, peak)},
        "per_event_protocol": {
            "api_ms": round(ms_ev_api, 4), "api_fused_option_ms": round(ms_ev_api_fused, 4),
            "fused_ms": round(ms_ev_fused, 4),
            "api_cells_per_s": round(ev / ms_ev_api * 1e3), "fused_cells_per_s": round(ev / ms_ev_fused * 1e3),
            "note": "one 436x436 event per rep from pinned AoS: copy_collection + calibrate + noise (api) or "
                    "transfer_calibrate (fused), host-synchronous; mean of the 10 fastest of 50 reps cycling "
                    "10 events (bench.py:214-289)"},
        "api_note": "api_*: copy_collection(per_field@cuda, aos) + funcs.calibrate_energy() + funcs.get_noise(), "
                    "the reference's prepare phase (bench.py:174-178): one conversion launch plus the two K5 "
                    "kernels, i.e. two more passes over the planes than the fused transfer_calibrate; "
                    "api_fused_option_*: the same three calls with copy_collection(..., {'fuse': 'sensor_funcs'}), "
                    "which runs the fused K1+K5 pass and leaves the behaviors nothing to do",
    }


def soakit_plugin_paths(a2, cells, dev, timed, noise_ref):
    """Config 2's prepare phase through soakit itself (baseline/_ref) with the plugin installed: soakit's
    copy_collection(per_field@cuda, aos@pinned) -> b200-convert, then soakit's coll.funcs.calibrate_energy() /
    get_noise() (the reference's bench.py:174-178 with cuda for mockdev). None when soakit is absent."""
    import numpy as np

    from oracle import cpu_baseline
    from paper_2511_04853_b200 import _native as nat

    soakit = cpu_baseline.import_reference()
    if soakit is None:
        return None
    from paper_2511_04853_b200 import soakit_plugin

    soakit_plugin.install()
    from soakit.detector import schemas as ds

    host = soakit.Collection(ds.SENSOR_SCHEMA, "aos", soakit_plugin.pinned_info())
    host.resize(cells)
    nat.memcpy(host.layout._struct_buf._data.ctypes.data, a2.layout._struct_buf.ptr, cells * 30, dev)
    nat.sync(dev)
    devc = soakit.Collection(ds.SENSOR_SCHEMA, "per_field", soakit_plugin.cuda_info(dev))

    def prepare():
        soakit.transfer.copy_collection(devc, host)
        with soakit.memctx.execution_scope("cuda"):
            devc.funcs.calibrate_energy()
            return devc.funcs.get_noise()

    ms = timed(prepare, steps=3, warmup=1)
    noise = prepare()
    # the same events through this package's own route: both noises must be the same bytes
    if np.asarray(noise).tobytes() != noise_ref.numpy().tobytes():
        raise SystemExit("config 2 through soakit: noise differs from the package route")
    return {"prepare_ms": round(ms, 3), "cells_per_s": round(cells / ms * 1e3),
            "h2d_gbs": round(cells * 30 / ms / 1e6, 1), "parity": "noise byte-equal to the package route",
            "note": "soakit 0.1.0 itself (baseline/_ref) + soakit_plugin.install(): copy_collection(per_field@cuda, "
                    "aos@pinned) + funcs.calibrate_energy() + funcs.get_noise(), 64 events per call. get_noise() "
                    "returns the reference's type, a host numpy array, so each call also moves 49 MB of noise "
                    "to the host (into page-locked memory recycled once the caller drops the array, "
                    "memctx.host_return_array); the package route (api_pinned_e2e_ms) keeps it on the device"}


def verify_aosoa_tiles(ao, n: int, fields, dev: int, seed: int = 4, samples: int = 32) -> str:
    """First, last and random AoSoA tiles vs oracle/restate.to_aosoa over the
    Track records restated from the splitmix image (seed 4, word 0)."""
    import numpy as np

    from oracle import restate
    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import workloads as wl

    lanes, tb = ao.lanes, ao.tile_bytes
    rng = np.random.default_rng(99)
    tiles = sorted({0, ao.ntiles - 1, *(int(x) for x in rng.integers(0, ao.ntiles, samples))})
    spec = [(f.leaf, f.dtype) for f in fields]
    got = np.empty(tb, np.uint8)
    for t in tiles:
        r0, r1 = t * lanes, min(n, (t + 1) * lanes)
        rec = restate.splitmix_image(seed, 0, r0 * 60, (r1 - r0) * 60).view(wl.TRACK_AOS_DTYPE)
        want = restate.to_aosoa(rec, spec, lanes, tb)
        nat.memcpy(got.ctypes.data, ao.buffer.ptr + t * tb, tb, dev)
        nat.sync(dev)
        if got.tobytes() != want:
            raise SystemExit(f"config 4: AoSoA tile {t} (T={lanes}) differs from the oracle")
    return f"{len(tiles)} tiles (first, last, random) byte-exact vs oracle/restate.to_aosoa"


def verify_sensor_events(coll, noise, dev: int, events) -> str:
    """Energy and noise of sampled events vs the oracle's event generator and
    case-study arithmetic (events.py:85-133, detector/schemas.py:29-41)."""
    import numpy as np

    from oracle import restate
    from paper_2511_04853_b200 import _native as nat

    n = 436 * 436
    e_ptr = coll.layout.plane_address(coll.plan.leaf("energy"))
    for e in events:
        ev = restate.generate_event(436, 436, seed=e, density=0.002)
        energy = restate.calibrate(ev["counts"], ev["parameter_A"], ev["parameter_B"])
        want_noise = restate.noise(energy, ev["noise_A"], ev["noise_B"], ev["noisy"])
        got_e, got_n = np.empty(n, np.float32), np.empty(n, np.float32)
        nat.memcpy(got_e.ctypes.data, e_ptr + e * n * 4, n * 4, dev)
        nat.memcpy(got_n.ctypes.data, noise.ptr + e * n * 4, n * 4, dev)
        nat.sync(dev)
        if got_e.tobytes() != energy.tobytes() or got_n.tobytes() != want_noise.tobytes():
            raise SystemExit(f"config 2: event {e} energy/noise differ from the oracle")
    return f"events {list(events)}: energy and noise bit-exact vs the oracle (generate_event + calibrate + noise)"


def _cfg_roofline(key: str, algo_bytes: float, ms: float, units: float, peak: float) -> dict:
    """roofline object of one config: algorithmic bytes per launch / launch time against the measured HBM
    peak, plus the DRAM bytes per launch ncu saw for this kernel (profiles/ncu_traffic.json, scaled to
    `units` of the workload's unit)."""
    achieved = algo_bytes / (ms / 1e3) / 1e9
    out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "traffic": None}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)["entries"][key]
        out["traffic"] = round(e["dram_bytes_per_unit"] * units)
        out["traffic_capture"] = e["capture"]
    except (OSError, KeyError, ValueError):
        pass
    return out


def _traffic(n: int):
    """dram bytes per launch from the committed ncu capture (profiles/), scaled to
    this launch's object count; None when no capture is committed."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return round(t["dram_bytes_per_object"] * n)
    except (OSError, KeyError, ValueError):
        return None


def run_extras(args, dev: int) -> dict:
    """Configs 1-4 on one GPU (device-resident inputs, CUDA-event timing)."""
    import numpy as np

    import paper_2511_04853_b200 as sk
    from paper_2511_04853_b200 import _native as nat
    from paper_2511_04853_b200 import jagged, layouts as ly, memctx as mc, schema as sc, sensor, transfer as tr
    from paper_2511_04853_b200 import workloads as wl
    from paper_2511_04853_b200.devarray import DeviceArray

    cuda = mc.ContextInfo.cuda(dev)
    peak = float(_peaks().get("hbm_gbs", 6650.0))

    def coll(schema, kind, n, info=cuda):
        c = sk.Collection(schema, kind, info)
        with mc.execution_scope(mc.CUDA if info.context == mc.CUDA else mc.HOST):
            c.reserve(n)
        with c.layout.engine_ops():
            c.layout._set_sizes_for_engine({sc.MAIN_TAG: n})
        return c

    def timed(fn, steps=5, warmup=2):
        for _ in range(warmup):
            fn()
        nat.sync(dev)
        a, b = nat.Event(), nat.Event()
        a.record(dev)
        for _ in range(steps):
            fn()
        b.record(dev)
        return a.elapsed_ms(b) / steps

    busy = DeviceArray(6 << 30, np.uint8, cuda)

    def queued(fn, steps=20, warmup=3):
        """device time of an asynchronous op: the launches are queued behind a
        ~1.5 ms device fill, so the event pair brackets GPU work only (small
        ops are otherwise bounded by the host's launch rate)"""
        for _ in range(warmup):
            fn()
        nat.sync(dev)
        a, b = nat.Event(), nat.Event()
        nat.call("sk_fill_random", busy.ptr, busy.n, 1, 0, nat.stream(dev))
        a.record(dev)
        for _ in range(steps):
            fn()
        b.record(dev)
        nat.sync(dev)
        return a.elapsed_ms(b) / steps

    out = {}
    # config 1: 1M Obj8 AoS -> SoA (launch-bound size), device-resident and from pinned host
    n = 1_000_000
    a1, p1 = coll(wl.OBJ8_SCHEMA, ly.AOS, n), coll(wl.OBJ8_SCHEMA, ly.PER_FIELD, n)
    wl.fill_random_device(a1.layout._struct_buf.ptr, n * 32, 1, dev)
    ms = queued(lambda: tr.copy_collection(p1, a1, {"async": True}), steps=20)
    # cold L2: rotate over 4 input/output pairs (256 MB > the 126 MB L2), so no conversion finds its
    # records or planes left in L2 by the previous one
    sets = [(a1, p1)]
    for k in range(3):
        a, p = coll(wl.OBJ8_SCHEMA, ly.AOS, n), coll(wl.OBJ8_SCHEMA, ly.PER_FIELD, n)
        wl.fill_random_device(a.layout._struct_buf.ptr, n * 32, 2 + k, dev)
        sets.append((a, p))
    turn = itertools.cycle(sets)

    def cold():
        a, p = next(turn)
        tr.copy_collection(p, a, {"async": True})

    ms_cold = queued(cold, steps=40)
    h1 = coll(wl.OBJ8_SCHEMA, ly.AOS, n, mc.ContextInfo.pinned())
    ms_h = timed(lambda: tr.copy_collection(p1, h1), steps=5)
    out["config1_obj8_1M"] = {"device_ms": round(ms, 4), "device_gbs": round(n * 64 / ms / 1e6, 1),
                              "frac": round(n * 64 / ms / 1e6 / peak, 3),
                              "cold_l2_device_ms": round(ms_cold, 4),
                              "cold_l2_frac": round(n * 64 / ms_cold / 1e6 / peak, 3),
                              "pinned_h2d_e2e_ms": round(ms_h, 3), "e2e_gbs": round(n * 64 / ms_h / 1e6, 1),
                              "note": "device_ms repeats one 64 MB pair (L2-resident: 64 MB < 126 MB L2); "
                                      "cold_l2 rotates 4 pairs (256 MB) so every launch reads and writes HBM",
                              "roofline": _cfg_roofline("config1_obj8_1M", n * 64, ms_cold, n, peak)}
    for a, p in sets:
        a.free()
        p.free()
    h1.free()

    # config 2: case study, 64 events x 190,096 cells generated on the device
    # (splitmix64, density 0.002), AoS (30 B) -> planes + energy + noise fused
    cells = 64 * 436 * 436
    gen = sk.Collection(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cuda)
    ms_gen = timed(lambda: sensor.generate_events(gen, 436, 436, range(64), 0.002, sync=False), steps=3, warmup=1)
    a2 = coll(sensor.SENSOR_SCHEMA, ly.AOS, cells)
    tr.copy_collection(a2, gen)  # K2: the events as the AoS records a host application would hold
    p2 = coll(sensor.SENSOR_SCHEMA, ly.PER_FIELD, cells)
    noise = DeviceArray(cells, np.float32, cuda)
    ms = queued(lambda: sensor.transfer_calibrate(p2, a2, noise, sync=False), steps=10)
    h2 = coll(sensor.SENSOR_SCHEMA, ly.AOS, cells, mc.ContextInfo.pinned())
    tr.copy_collection(h2, a2)
    ms_h = timed(lambda: sensor.transfer_calibrate(p2, h2, noise, sync=True), steps=3, warmup=1)
    out["config2_sensor_64x190096"] = {
        "device_ms": round(ms, 3), "device_cells_per_s": round(cells / ms * 1e3),
        "device_gbs": round(cells * 64 / ms / 1e6, 1), "frac": round(cells * 64 / ms / 1e6 / peak, 3),
        "pinned_h2d_e2e_ms": round(ms_h, 3), "e2e_cells_per_s": round(cells / ms_h * 1e3),
        "h2d_gbs": round(cells * 30 / ms_h / 1e6, 1),
        "event_generation_ms": round(ms_gen, 3), "event_generation_cells_per_s": round(cells / ms_gen * 1e3),
        "data": "64 events 436x436, seeds 0..63, density 0.002, generated on-device (bit-exact with "
                "detector/events.py:85-133)"}
    out["config2_sensor_64x190096"]["roofline"] = _cfg_roofline("config2_sensor_fused", cells * 64, ms, cells, peak)
    out["config2_sensor_64x190096"]["parity"] = verify_sensor_events(p2, noise, dev, (0, 31, 63))
    out["config2_sensor_64x190096"].update(config2_api_paths(a2, p2, h2, noise, cells, dev, peak, queued, timed))
    out["config2_sensor_64x190096"]["parity_api_path"] = verify_sensor_events(p2, noise, dev, (5, 47))
    sp = soakit_plugin_paths(a2, cells, dev, timed, noise)
    if sp is not None:
        out["config2_sensor_64x190096"]["through_soakit"] = sp
    # the reference's second phase on the same events: reconstruct + transfer back (bench.py:180-184)
    from paper_2511_04853_b200 import sensor as sn

    sn.calibrate_collection(p2)
    parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, cuda)
    ms_r = timed(lambda: sn.reconstruct_from_collection(p2, 436, 436, out=parts, events=64, noise=noise),
                 steps=3, warmup=1)
    host_parts = sk.Collection(sensor.PARTICLE_SCHEMA, ly.PER_FIELD, mc.ContextInfo.pinned())
    ms_rt = timed(lambda: (sn.reconstruct_from_collection(p2, 436, 436, out=parts, events=64, noise=noise),
                           tr.copy_collection(host_parts, parts)), steps=3, warmup=1)
    # ... and the reference's export of the result (bench.py:180-184 -> baselines.py:104-120): K2 into packed
    # particle records on the device, one D2H per buffer, the records + per-particle sensor lists on the host
    stage = sk.Collection(sensor.PARTICLE_SCHEMA, ly.AOS, mc.ContextInfo.pinned())
    ms_ex = timed(lambda: (sn.reconstruct_from_collection(p2, 436, 436, out=parts, events=64, noise=noise),
                           sn.export_particles_from_collection(parts, stage)), steps=3, warmup=1)
    out["config2_reconstruct_64_events"] = {
        "ms": round(ms_r, 3), "events_per_s": round(64 / ms_r * 1e3), "particles": len(parts),
        "rounds": parts.reco_rounds, "with_transfer_back_ms": round(ms_rt, 3),
        "with_export_ms": round(ms_ex, 3),
        "note": "round-synchronous parallel greedy, same particles/order as reconstruct_arrays; with_export: "
                "+ export_particles_from_collection (PARTICLE_AOS_DTYPE records and sensor lists on the host)"}
    for c in (a2, p2, h2, gen, parts, host_parts, stage):
        c.free()
    noise.free()

    # config 3: 1M clusters, ~10M u64 members, shuffled source pool
    nc = 1_000_000
    lens, offsets, pool = wl.cluster_inputs(nc, seed=7)
    d_lens, d_off, d_pool = DeviceArray.from_numpy(lens, cuda), DeviceArray.from_numpy(offsets, cuda), \
        DeviceArray.from_numpy(pool, cuda)
    c3 = sk.Collection(wl.CLUSTER_SCHEMA, ly.PER_FIELD, cuda)
    with mc.execution_scope(mc.CUDA):
        c3.resize(nc)
    members = int(lens.sum())
    ms_api = timed(lambda: jagged.pack(c3, "members", d_lens, d_off, d_pool), steps=10)
    # the same call with the inputs in pinned and in pageable HOST memory: validation on the host, the
    # H2D of lengths / offsets / pool and the pack, with the member total read back
    pinned_in = []
    for x in (lens, offsets, pool):
        b = mc.allocate(mc.ContextInfo.pinned(), x.nbytes)
        v = b._data.view(x.dtype)
        v[:] = x
        pinned_in.append((b, v))
    ms_pinned = timed(lambda: jagged.pack(c3, "members", *(v for _, v in pinned_in)), steps=5, warmup=1)
    ms_pageable = timed(lambda: jagged.pack(c3, "members", lens, offsets, pool), steps=3, warmup=1)
    for b, _ in pinned_in:
        mc.deallocate(b)
    # the reference's own API: Collection.jagged_fill(path, segments) with one numpy vector per record
    # (collection.py:537-556), the vectors being views into the shuffled source pool
    segments = [pool[o:o + k] for o, k in zip(offsets.tolist(), lens.tolist())]
    ms_fill = timed(lambda: c3.jagged_fill("members", segments), steps=5, warmup=2)
    with mc.execution_scope(mc.CUDA):
        fill_p, fill_m = c3.prefix_sums("members"), c3.column("members").read()
    del segments
    # the same fused pack through the C-ABI (scan + gather, no host readback), device time
    import ctypes as C

    i32 = nat.TYPE_CODES["i32"]
    prefix = DeviceArray(nc + 1, np.int32, cuda)
    cap = members + 4096
    need = C.c_size_t(0)
    nat.call("sk_jagged_scratch_bytes", nc, C.byref(need))
    scratch = DeviceArray(-(-need.value // 256) * 256 + ((cap + 255) // 256 + 1) * 8, np.uint8, cuda)
    total = DeviceArray(2, np.int64, cuda)
    pool_out = DeviceArray(cap, np.uint64, cuda)
    foff, fsz, dst = (C.c_int64 * 1)(0), (C.c_int32 * 1)(8), (C.c_void_p * 1)(pool_out.ptr)
    strm = nat.stream(dev)
    ms = queued(lambda: nat.call("sk_jagged_pack", nc, d_lens.ptr, i32, prefix.ptr, i32, d_off.ptr, d_pool.ptr,
                                 pool.size, 8, 1, foff, fsz, dst, cap, scratch.ptr, scratch.n, total.ptr, strm),
                steps=20)
    algo = nc * 16 + members * 16
    from oracle import restate

    want_p, want_m = restate.jagged_pack(lens, offsets, pool, np.int32)
    if prefix.numpy().tobytes() != want_p.tobytes() or pool_out.numpy()[:members].tobytes() != want_m.tobytes():
        raise SystemExit("config 3: packed prefix/pool differ from the oracle")
    if np.asarray(fill_p).tobytes() != want_p.tobytes() or np.asarray(fill_m).tobytes() != want_m.tobytes():
        raise SystemExit("config 3: jagged_fill prefix/pool differ from the oracle")
    out["config3_jagged_1M"] = {
        "members": members, "device_ms": round(ms, 4), "members_per_s": round(members / ms * 1e3),
        "gbs": round(algo / ms / 1e6, 1), "frac": round(algo / ms / 1e6 / peak, 3),
        "api_ms": round(ms_api, 4),
        "jagged_fill": {"ms": round(ms_fill, 3), "members_per_s": round(members / ms_fill * 1e3),
                        "gbs": round(algo / ms_fill / 1e6, 2),
                        "note": "Collection.jagged_fill('members', segments), segments = 1M numpy views into the "
                                "shuffled host pool (the reference's call, collection.py:537-556): threaded C "
                                "packing into pinned staging, one H2D, the fused pack; prefix and pool checked "
                                "byte-exact vs the oracle"},
        "host_input_e2e": {"pinned_ms": round(ms_pinned, 3), "pageable_ms": round(ms_pageable, 3),
                           "h2d_bytes": int(lens.nbytes + offsets.nbytes + pool.nbytes),
                           "note": "jagged.pack(collection, lens, offsets, pool) with numpy inputs in pinned / "
                                   "pageable host memory: host-side validation (collection.py:546 raises before "
                                   "mutating), H2D of the inputs, the fused pack, member total read back"},
        "note": "device_ms: sk_jagged_pack queued on the device: one launch of pack_reg_kernel (1792-record tiles, "
                "decoupled look-back for the prefix, register gather); api_ms: jagged.pack on a Collection, incl. "
                "the host readback of the member total and invalid-segment count; source segments in shuffled "
                "order with slack: ncu counts 133 MB of DRAM reads for 92 MB of algorithmic reads "
                "(64-byte fetch granularity, profiles/r02_jagged_redesign.md)",
        "parity": "whole prefix (1,000,001 x i32) and pool byte-exact vs oracle/restate.jagged_pack",
        "roofline": _cfg_roofline("config3_jagged_1M", algo, ms, 1, peak)}
    c3.free()
    for d in (d_lens, d_off, d_pool, prefix, scratch, total, pool_out):
        d.free()

    # config 3 at 10M clusters (~100M members): the same fused pack, the whole prefix and 4096 sampled
    # records' members checked against the numpy restatement
    n10 = 10_000_000
    lens, offsets, pool = wl.cluster_inputs(n10, seed=8)
    d_lens, d_off, d_pool = (DeviceArray.from_numpy(x, cuda) for x in (lens, offsets, pool))
    members = int(lens.sum())
    prefix = DeviceArray(n10 + 1, np.int32, cuda)
    cap = members + 4096
    nat.call("sk_jagged_scratch_bytes", n10, C.byref(need))
    scratch = DeviceArray(-(-need.value // 256) * 256, np.uint8, cuda)
    total = DeviceArray(2, np.int64, cuda)
    pool_out = DeviceArray(cap, np.uint64, cuda)
    dst = (C.c_void_p * 1)(pool_out.ptr)
    ms = queued(lambda: nat.call("sk_jagged_pack", n10, d_lens.ptr, i32, prefix.ptr, i32, d_off.ptr, d_pool.ptr,
                                 pool.size, 8, 1, foff, fsz, dst, cap, scratch.ptr, scratch.n, total.ptr, strm),
                steps=10)
    algo = n10 * 16 + members * 16
    want_p = np.concatenate([[0], np.cumsum(lens, dtype=np.int64)]).astype(np.int32)
    got_p = prefix.numpy()
    ok = got_p.tobytes() == want_p.tobytes() and total.numpy().tolist() == [members, 0]
    sample = np.random.default_rng(9).integers(0, n10, 4096)
    got_m = pool_out.numpy()
    for r in sample.tolist():
        a, k, o = int(want_p[r]), int(lens[r]), int(offsets[r])
        ok = ok and got_m[a:a + k].tobytes() == pool[o:o + k].tobytes()
    if not ok:
        raise SystemExit("config 3 at 10M clusters: prefix or sampled members differ from the restatement")
    out["config3_jagged_10M"] = {
        "members": members, "device_ms": round(ms, 4), "members_per_s": round(members / ms * 1e3),
        "gbs": round(algo / ms / 1e6, 1), "frac": round(algo / ms / 1e6 / peak, 3),
        "parity": "whole prefix (10,000,001 x i32) and the members of 4096 random records byte-exact vs the "
                  "numpy restatement (cumsum, pool slices)",
        "roofline": _cfg_roofline("config3_jagged_10M", algo, ms, 1, peak)}  # no capture: traffic null
    for d in (d_lens, d_off, d_pool, prefix, scratch, total, pool_out):
        d.free()

    # config 4: 100M Track records (60 B) -> AoSoA T=128 of [pz, px, x, charge] with f64->f32
    n4 = 100_000_000
    a4 = coll(wl.TRACK_SCHEMA, ly.AOS, n4)
    wl.fill_random_device(a4.layout._struct_buf.ptr, n4 * 60, 4, dev)
    fields = [sk.AosoaField("pz", "f32"), sk.AosoaField("px", "f32"), sk.AosoaField("x", "f32"),
              sk.AosoaField("charge", "i32")]
    ao = sk.Aosoa(n4, 128, fields, cuda)
    ms = queued(lambda: sk.to_aosoa(a4, fields, 128, out=ao, sync=False), steps=10)
    out["config4_aosoa_100M"] = {"ms": round(ms, 3), "gbs": round(n4 * 76 / ms / 1e6, 1),
                                 "frac": round(n4 * 76 / ms / 1e6 / peak, 3), "objects_per_s": round(n4 / ms * 1e3)}
    out["config4_aosoa_100M"]["roofline"] = _cfg_roofline("config4_aosoa_100M", n4 * 76, ms, n4, peak)
    out["config4_aosoa_100M"]["parity"] = verify_aosoa_tiles(ao, n4, fields, dev)
    ao.free()
    # the other tile widths SURVEY 8d names (T = 32, 64): same bytes per object
    for lanes in (32, 64):
        ao = sk.Aosoa(n4, lanes, fields, cuda)
        ms = queued(lambda: sk.to_aosoa(a4, fields, lanes, out=ao, sync=False), steps=5)
        out["config4_aosoa_100M"][f"T{lanes}"] = {"ms": round(ms, 3), "gbs": round(n4 * 76 / ms / 1e6, 1),
                                                  "frac": round(n4 * 76 / ms / 1e6 / peak, 3),
                                                  "parity": verify_aosoa_tiles(ao, n4, fields, dev, samples=8)}
        ao.free()
    # the same conversion from HOST records: a 16M-track pinned sample through the API, the H2D chunked
    # and overlapped with the conversion on the device (first and last tiles checked)
    nh = 16_000_000
    h4 = coll(wl.TRACK_SCHEMA, ly.AOS, nh, mc.ContextInfo.pinned())
    nat.memcpy(h4.layout._struct_buf._data.ctypes.data, a4.layout._struct_buf.ptr, nh * 60, dev)
    nat.sync(dev)
    ao = sk.Aosoa(nh, 128, fields, cuda)
    ms_h = timed(lambda: sk.to_aosoa(h4, fields, 128, out=ao), steps=5, warmup=1)
    out["config4_aosoa_100M"]["host_input_e2e"] = {
        "objects": nh, "ms": round(ms_h, 3), "objects_per_s": round(nh / ms_h * 1e3),
        "gbs": round(nh * 76 / ms_h / 1e6, 1), "h2d_gbs": round(nh * 60 / ms_h / 1e6, 1),
        "h2d_bytes": nh * 60, "parity": verify_aosoa_tiles(ao, nh, fields, dev, samples=4),
        "note": "to_aosoa(pinned Track AoS collection, fields, 128, out=device Aosoa): the host records go "
                "over the link in chunks overlapped with the AoSoA conversion on the device; gbs counts the "
                "same 76 algorithmic bytes per object as the device-resident line"}
    ao.free()
    h4.free()
    a4.free()
    busy.free()
    return out


# ---- the reference arm -----------------------------------------------------------------------------

def run_reference(args) -> None:
    rank, world, _ = _dist()
    if rank != 0:
        return
    from oracle import cpu_baseline

    procs = os.cpu_count() or 1
    n = args.ref_objects
    r = cpu_baseline.reference_multi_core(n, args.steps, max(1, args.warmup), procs)
    if r is not None:
        what = (f"soakit's own copy_collection(per_field, aos) (per-leaf-default, transfer.py:171-236) from "
                f"baseline/_ref, one process per core, each owning 1/{procs} of the records")
    else:
        r = dict(cpu_baseline.multi_core(n, args.steps, max(1, args.warmup), procs), kind="port")
        what = f"reference per-leaf numpy path (oracle/cpu_baseline.py) sharded over {procs} processes"
    times = r["step_seconds"]
    t = statistics.mean(times)
    value = n * BYTES_PER_OBJECT / t / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (random Obj8 records)", "impl": "reference",
        "config": {"workload": WORKLOAD, "objects_per_step": n, "record_bytes": 32,
                   "algorithmic_bytes_per_object": BYTES_PER_OBJECT,
                   "sample_note": f"each step converts a bounded {n}-object sample of the 1e9-object workload "
                                  "(the CPU would need minutes per full step); the metric is a rate (GB/s), "
                                  "compared rate against rate with our arm"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": procs, "kind": r["kind"],
                         "sample": f"{n} Obj8 objects per step, {what}; host: {_cpu_info()}"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--objects", type=int, default=1_000_000_000)
    ap.add_argument("--e2e-objects", type=int, default=64_000_000)
    ap.add_argument("--cpu-objects", type=int, default=16_000_000)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-objects", type=int, default=64_000_000)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-p2p", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
