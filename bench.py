#!/usr/bin/env python
"""bench.py -- Mkeys/s of the B200 adaptive sort on BASELINE.json's workloads.

Default line (N=1): configs[1] ("c2"): n = 2,000,000 int32 keys, four orders
(random, reversely sorted, nearly sorted = n/100 swaps, few unique = 10
values).  One STEP = one sort of one instance of each of the four orders
(8,000,000 keys); value = keys sorted / summed device time of the sorts.  The
same line carries, under "c5a", configs[4]'s 256M-key int32 random sort (the
metric's "n=2M/256M" second half), measured the same way in the same run.

Timing: every sort is bracketed by CUDA events on the sort's stream.  No sort
finds its input in L2.  The 2M-key workloads run configs[1]'s procedure --
seeded instances of each order sorted back to back -- with one input buffer
per sort of the run (steps + warmup, every order: 736 MB by default, >= 4 L2
sizes or the flush below is used), all restored from pristine copies before
the first sort, so every input comes from HBM while what the sorts share (the
kernels' code, the scratch) stays cached; detail.l2_flushed times a few steps
the other way: input restored and L2 flushed by a 512 MiB write before every
sort (untimed), which also evicts the code.  The 1 GiB workloads (one instance
per order) use the flush.  The K timed steps are bracketed by barrier +
synchronize on both sides and the max over ranks is taken.  e2e: the same metric through the host-buffer calls (HOST
pinned buffers; H2D copies, sorts, D2H copies and the stream sync inside the
events): the step's instances as one sr_sort_host_batch call (uploads and
downloads of neighbouring instances overlap the sorts), with the
one-sr_sort_host-call-per-instance figure under "per_call"; single-instance
workloads use sr_sort_host.

Every timed output is checked after the timed region: on rank 0 at N=1 the
cpu_baseline leg runs the oracle (single-threaded, pinned to one core) on the
very instances the GPU sorted and compares bit for bit; elsewhere the output is
checked on the device by properties (sorted, multiset fingerprints, payload
invariants).  A failed check exits non-zero.

--impl reference runs the CPU oracle (the reference arm for this tier: a plain
single-threaded mergesort, oracle/) on a bounded sample of the same workload,
and prints the same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import gen  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# BASELINE.json metric, printed verbatim by both arms (the driver pairs them on it)
METRIC = "Mkeys/s sorted (int32, n=2M/256M, 4 input types); achieved HBM GB/s vs peak"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback

WORKLOADS = {
    # name: (n, dtype, orders, config index for seeds)
    "c2": (2_000_000, np.int32, ["random", "reversed", "nearly", "few_unique"], 1),
    "c1": (1_000_000, np.int32, ["random"], 0),
    "c5a": (268_435_456, np.int32, ["random"], 4),
    "c5b": (268_435_456, np.int32, ["nearly1000"], 4),
    "c5c": (134_217_728, np.int64, ["random"], 4),
    "c3": (16_777_216, np.int32, ["swaps_1e4", "swaps_1e3", "swaps_1e2", "swaps_1e1", "runs1024", "last1pct",
                                  "alternating"], 2),
    "c4": (16_777_216, np.int32, ["few100"], 3),  # stable key-value sort, payload = original index
    # report-only widenings: the paper's "random
    # double" and "random 16-list" classes at the Table 1 size
    "c2d": (2_000_000, np.float64, ["funiform", "fbits"], 1),
    "c2l16": (2_000_000, ("rec", 16), ["lrandom", "lprefix"], 1),
    "c2l256": (200_000, ("rec", 256), ["lrandom", "lprefix"], 1),  # the paper's 256-int lists (1024 B)
    # report-only: the paper's Table 1 "nearly sorted" class is 256-distance
    # (PAPER.md:36, :84); configs[1](c) uses k-exchange instead
    "c2k": (2_000_000, np.int32, ["distance256"], 1),
    "c3k": (16_777_216, np.int32, ["distance256"], 2),
}


PAIRS = {"c4"}  # workloads sorted as (key, payload = original index) pairs


def is_rec(dtype):
    return isinstance(dtype, tuple)


def elem_bytes(dtype):
    return 4 * dtype[1] if is_rec(dtype) else np.dtype(dtype).itemsize


def dtype_label(dtype):
    if is_rec(dtype):
        return f"i32x{dtype[1]}"
    return {"int32": "i32", "int64": "i64", "float32": "f32", "float64": "f64"}[np.dtype(dtype).name]


def oracle_sort(a, pairs=False):
    import oracle
    if pairs:  # payload = original index (configs[3])
        return oracle.sort_pairs(a, gen.index_payload(a.size))
    return oracle.sort_records(a) if a.ndim == 2 else oracle.sort_keys(a)


def make_input(order, n, dtype, config, instance):
    if order == "nearly1000":
        return gen.swaps(n, n // 1000, dtype, gen.seed_for(config, 2, instance))
    if is_rec(dtype):
        return gen.make_list(order, n, dtype[1], config=config, instance=instance)
    if np.dtype(dtype).kind == "f":
        return gen.make_float(order, n, dtype, config=config, instance=instance)
    return gen.make(order, n, dtype, config=config, instance=instance)


def make_input_dev(sr, order, n, dtype, config, instance, dev):
    """The same input as make_input, generated on the device by sr_generate
    (random and swap orders of integer keys), else None."""
    import torch
    if is_rec(dtype) or np.dtype(dtype).kind != "i":
        return None
    t = torch.empty(n, dtype=torch.int32 if np.dtype(dtype) == np.int32 else torch.int64, device=dev)
    if order == "random":
        sr.generate(t, "random", gen.seed_for(config, gen.ORDERS["random"], instance))
    elif order == "nearly1000":
        sr.generate(t, "swaps", gen.seed_for(config, 2, instance), n // 1000)
    elif order == "distance256":
        sr.generate(t, "distance", gen.seed_for(config, gen.ORDERS[order], instance), 256)
    else:
        return None
    return t


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled every ~0.5 ms during the timed region
    (NVML in-process; the timed region is far shorter than nvidia-smi's -lms
    floor).  Falls back to one nvidia-smi query if NVML is unavailable."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index=0):
        self.index = index
        self.sm = []
        self.reasons = set()
        self.max_mhz = None
        self.stop = threading.Event()
        self.t = None
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def sample_now(self):
        """One sample from the calling thread (the timed loop calls it between two sorts, outside
        their events: the sampler thread rarely gets scheduled inside a ~6 ms region)."""
        nv = self.nv
        if nv is None:
            return
        try:
            self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, attr in self.REASONS.items():
                if r & getattr(nv, attr, 0):
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self.stop.is_set():
            self.sample_now()
            time.sleep(0.0005)

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=1)

    def absorb(self, other):
        """Add the samples of another window of timed sorts (the flushed variant, the e2e passes)."""
        self.extra = getattr(self, "extra", 0) + len(other.sm)
        self.sm += other.sm
        self.reasons |= other.reasons
        self.max_mhz = self.max_mhz or other.max_mhz

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        extra = getattr(self, "extra", 0)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "sm_mhz_min": min(self.sm),
                "windows": f"{len(self.sm) - extra} samples during the K timed steps, {extra} during the other timed "
                           "sorts of the run (flushed variant, e2e passes)"}


# bench kernel names (sr_last_profile) -> ncu kernel-name prefixes
NCU_NAMES = {"presort_scan": "k_presort_scan", "presort_resolve": "k_presort_resolve", "reverse": "k_reverse",
             "sample_rank": "k_sample_rank", "select_splitters": "k_select_splitters", "count": "k_count",
             "plan": "k_plan", "scatter": "k_scatter", "finish_small": "k_finish_warp", "finish": "k_finish<",
             "merge": "k_merge<", "scan": "k_scan_u32", "resident": "k_resident"}


def ncu_traffic(kernel: str, dtype_name: str, workload: str):
    """DRAM read+write bytes per launch of `kernel` from the newest committed
    ncu --set full summary of the same workload (profiles/*_ncu_summary.json,
    "workload" field), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json")))  # tags sort by round/session (r1_ < r1s2 < r1s3 < r1s3f < r1s4); mtimes do not survive a checkout
    pref = NCU_NAMES.get(kernel)
    for f in reversed(files):
        try:
            summ = json.load(open(f))
        except Exception:
            continue
        if summ.get("workload") != workload:
            continue
        full = summ.get("full", {})
        for name, d in full.items():
            if pref and name.startswith(pref) and f"<{dtype_name}" in name.replace(" ", ""):
                r, w = d.get("dram_bytes_read") or 0, d.get("dram_bytes_write") or 0
                return {"bytes": int(r + w), "source": os.path.relpath(f, ROOT), "ncu_kernel": name}
    return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def instance_ids(rank: int, per_rank: int) -> list:
    """Weak scaling over independent problems: rank r sorts its own instances
    r*per_rank .. r*per_rank+per_rank-1 (no data-path collective)."""
    return [rank * per_rank + i for i in range(per_rank)]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank time over all ranks (1 rank: identity)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def pin_one_core():
    """Pin this process to one host core for the oracle legs;
    returns (restore-set, core) or (None, None) where affinity is unsupported."""
    try:
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
        return old, core
    except Exception:
        return None, None


def unpin(old):
    if old:
        try:
            os.sched_setaffinity(0, old)
        except Exception:
            pass


L2_BYTES = 126 * 1024 * 1024
L2_TEXT = {
    "flush": "flushed (512 MiB write) before every sort, outside the timed region",
    "rotate": "inputs larger than L2: every sort of the run (steps + warmup, every order) has its own input "
              "buffer, all restored from the pristine instances before the first sort, so at least 4x the L2 "
              "size of other traffic lies between an input's last write and its sort (the input comes from HBM; "
              "what the sorts share -- code, scratch -- stays cached, as between the paper's 100 instances per "
              "order); the flushed variant is under detail.l2_flushed",
}


def l2_mode(wl, args):
    """How the timed sorts are kept from finding their input in L2: "rotate"
    (distinct input buffers, >= 4 L2 sizes in total; configs[1]'s "100 seeded
    instances each of four input orders" back to back) when the run's inputs
    are that large, else "flush" (a 512 MiB write before every sort; this also
    evicts the kernels' code, which the next sort then fetches from HBM).  The
    1 GiB workloads sort one instance per order: flush."""
    n, dtype, orders, cfg = WORKLOADS[wl]
    per = n * (elem_bytes(dtype) + (4 if wl in PAIRS else 0))
    if args.l2 == "flush" or n >= 50_000_000:
        return "flush"
    return "rotate" if per * len(orders) * (args.steps + args.warmup) >= 4 * L2_BYTES else "flush"


def ref_config(wl, args):
    """The workload description both arms print (the driver pairs the arms on
    metric + config)."""
    n, dtype, orders, cfg = WORKLOADS[wl]
    return {"workload": wl, "n": n, "dtype": dtype_label(dtype), "pairs": wl in PAIRS, "orders": orders,
            "keys_per_step": n * len(orders), "l2": L2_TEXT[l2_mode(wl, args)]}


def run_reference(args, wl):
    """Reference arm: the CPU oracle on a bounded sample of the workload."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n, dtype, orders, cfg = WORKLOADS[wl]
    budget = float(os.environ.get("SR_REF_BUDGET_S", "20"))
    # bounded sample: the first `m` keys of each order's instance, m chosen so a step is ~budget/(steps+warmup) s
    per_step = budget / max(1, args.steps + args.warmup)
    m = min(n, max(10_000, int(per_step / (len(orders) * 1.2e-7))))  # ~120 ns/key oracle estimate
    inputs = [make_input(o, n, dtype, cfg, 0)[:m].copy() for o in orders]
    old, core = pin_one_core()
    try:
        for _ in range(args.warmup):
            for a in inputs:
                oracle_sort(a, wl in PAIRS)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for a in inputs:
                oracle_sort(a, wl in PAIRS)
        dt = (time.perf_counter() - t0) / args.steps
    finally:
        unpin(old)
    keys = m * len(orders)
    v = keys / dt / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3),
            "unit": "Mkeys/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype_label(dtype), "data": "synthetic", "config": ref_config(wl, args),
            "cpu_baseline": {"value": round(v, 3), "unit": "Mkeys/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {m} keys of instance 0 of each order, single-threaded C mergesort"
                                       + (f" pinned to core {core}" if core is not None else "")},
            "e2e": {"value": round(v, 3), "unit": "Mkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- output checks
def _fp_dev(t):
    """Two commutative 64-bit fingerprints of a device tensor's multiset of
    bit patterns (wrapping int64 arithmetic; same function on input and output)."""
    import torch
    x = t.reshape(-1)
    x = x.view(torch.int32).to(torch.int64) if x.element_size() == 4 else x.view(torch.int64)
    h1 = (x * -7046029254386353131) ^ (x >> 29)
    h2 = (x ^ -2889434331225346157) * -6884282663029091281
    return int(h1.sum()), int(h2.sum())


def _total_order_image(t):
    """Signed-integer image of float keys in IEEE totalOrder (test-side check)."""
    import torch
    if t.dtype == torch.float32:
        b = t.view(torch.int32)
        return b ^ ((b >> 31) & 0x7FFFFFFF)
    if t.dtype == torch.float64:
        b = t.view(torch.int64)
        return b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFF)
    return t


def check_props(out_k, in_k, out_v=None, in_v=None):
    """Properties every correct output has, checked on the device (used where
    the oracle does not run: ranks > 0, N > 1, --no-cpu-baseline): keys
    non-decreasing (totalOrder for floats), same multiset as the input; for
    pairs with payload = original index: out_key == in_key[out_val], the
    payload a permutation, and increasing among equal keys (stability)."""
    import torch
    if out_k.dim() == 2:  # records: multiset only (the oracle leg checks order)
        return _fp_dev(out_k) == _fp_dev(in_k)
    img = _total_order_image(out_k)
    if img.numel() > 1 and not bool((img[1:] >= img[:-1]).all()):
        return False
    if _fp_dev(out_k) != _fp_dev(in_k):
        return False
    if out_v is not None:
        vi = out_v.view(torch.int32).to(torch.int64)
        if not torch.equal(out_k, in_k[vi]):
            return False
        if not torch.equal(torch.sort(vi).values, torch.arange(vi.numel(), device=vi.device)):
            return False
        same = out_k[1:] == out_k[:-1]
        if not bool((vi[1:] > vi[:-1])[same].all()):
            return False
    return True


# ----------------------------------------------------------------------------- one workload
def measure(wl, args, sr, dev, stream, rank, ws, oracle_leg):
    """Time K steps of workload `wl` (one step = one sort of one instance of
    each order), then e2e through the host API, a per-kernel profile pass, and
    the output checks.  Returns the fields of a bench line."""
    import torch
    n, dtype, orders, cfg = WORKLOADS[wl]
    rec = is_rec(dtype)
    pairs = wl in PAIRS
    tdt = torch.int32 if rec else {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32,
                                   "float64": torch.float64}[np.dtype(dtype).name]
    kw = elem_bytes(dtype) + (4 if pairs else 0)  # bytes per element (key + payload)
    shape = (n, dtype[1]) if rec else (n,)
    steps, warm = args.steps, args.warmup

    # inputs: instance = rank * (steps+warmup) + step  (weak scaling: independent problems per rank);
    # 1 GiB workloads sort one instance per order every step
    total = steps + warm
    big = n >= 50_000_000
    ninst = 1 if big else total
    pristine, host_inputs = {}, {}
    ids = instance_ids(rank, total)
    for o in orders:
        for i in range(ninst):
            t = make_input_dev(sr, o, n, dtype, cfg, ids[i], dev) if big else None
            if t is not None:  # 1 GiB inputs: built on the device (sr_generate, bit-identical to gen.py)
                pristine[(o, i)] = t
                host_inputs[(o, i)] = t.cpu().numpy()
                continue
            a = make_input(o, n, dtype, cfg, ids[i])
            pristine[(o, i)] = torch.from_numpy(a).to(dev)
            host_inputs[(o, i)] = a
    work = torch.empty(shape, dtype=tdt, device=dev)
    if pairs:  # configs[3]: payload = each element's original index (int32)
        vals_pristine = torch.from_numpy(gen.index_payload(n).view(np.int32)).to(dev)
        work_v = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    rotate = l2_mode(wl, args) == "rotate"
    works, works_v = {}, {}
    if rotate:  # one input buffer per sort of the run (see l2_mode)
        for i in range(total):
            for o in orders:
                works[(o, i)] = torch.empty(shape, dtype=tdt, device=dev)
                if pairs:
                    works_v[(o, i)] = torch.empty(n, dtype=torch.int32, device=dev)

    def restore_all():  # in the order the sorts run
        for i in range(total):
            for o in orders:
                works[(o, i)].copy_(pristine[(o, i % ninst)])
                if pairs:
                    works_v[(o, i)].copy_(vals_pristine)

    def one_sort(o, i, ev=None, flushed=False):
        """Sort instance i of order o; returns (plan, keys, vals) -- the buffers hold the output."""
        if rotate and not flushed:
            wk, wv = works[(o, i)], works_v.get((o, i))
        else:
            wk, wv = work, work_v if pairs else None
            wk.copy_(pristine[(o, i % ninst)])
            if pairs:
                wv.copy_(vals_pristine)
            flush.fill_(i)
        if ev:
            ev[0].record(stream)
        if rec:
            sr.sort_records(wk)
        elif pairs:
            sr.sort_pairs(wk, wv)
        else:
            sr.sort_keys(wk)
        if ev:
            ev[1].record(stream)
        return sr.last_plan(), wk, wv

    if rotate:
        restore_all()
    for w in range(warm):
        for o in orders:
            one_sort(o, w)
    torch.cuda.synchronize()

    # ---- timed region (outputs kept, untimed, for the checks after it)
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in orders]
           for _ in range(steps)]
    plans = []
    kept = {}          # small workloads: every timed output, on the device
    first_big = {}     # big workloads: the first timed output per order; later ones compared to it
    big_same = True
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        t_wall0 = time.perf_counter()
        for s in range(steps):
            if not big:
                clk.sample_now()  # (between two sorts, outside their events)
            for j, o in enumerate(orders):
                plan, wk, wv = one_sort(o, warm + s, evs[s][j])
                plans.append((o, plan))
                if big:
                    if o not in first_big:
                        first_big[o] = (wk.clone(), wv.clone() if pairs else None)
                    else:
                        big_same &= torch.equal(first_big[o][0], wk) and (not pairs or torch.equal(first_big[o][1], wv))
                elif rotate:
                    kept[(o, warm + s)] = (wk, wv)  # (the sort's own buffer: nothing else writes it before the checks)
                else:
                    kept[(o, warm + s)] = (wk.clone(), wv.clone() if pairs else None)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    if ws > 1:
        torch.distributed.barrier()
    per_order_ms = {o: [evs[s][j][0].elapsed_time(evs[s][j][1]) for s in range(steps)] for j, o in enumerate(orders)}
    step_ms = [sum(evs[s][j][0].elapsed_time(evs[s][j][1]) for j in range(len(orders))) for s in range(steps)]
    total_ms = max_over_ranks(sum(step_ms), dev)
    keys_all = n * len(orders) * steps * ws
    value = keys_all / (total_ms / 1e3) / 1e6
    launches = sum(p["launches"] for _, p in plans)
    bytes_planned = sum(p["bytes_planned"] for _, p in plans) / steps
    route_of = {o: p["route_name"] for o, p in plans[:len(orders)]}

    # ---- output checks (untimed): exact against the oracle in the oracle leg, properties elsewhere
    check = {"checked": 0, "failed": 0, "how": ""}
    cpu = None
    if big:
        to_check = [(o, 0, first_big[o]) for o in orders]
        check["repeat_identical"] = bool(big_same)
    else:
        to_check = [(o, idx, kept[(o, idx)]) for (o, idx) in kept]
    if oracle_leg:
        # the cpu_baseline leg: the oracle, single-threaded and pinned to one core,
        # sorts the very instances the GPU sorted (bounded: <= ~30 s of host work);
        # its outputs are the expected values of the exact comparison
        old, core = pin_one_core()
        t_sort, keys_done, n_sorts = 0.0, 0, 0
        budget = float(os.environ.get("SR_ORACLE_BUDGET_S", "30"))
        try:
            for (o, idx, (gk, gv)) in to_check:
                if t_sort > budget:
                    break
                a = host_inputs[(o, idx % ninst)]
                t0 = time.perf_counter()
                exp = oracle_sort(a, pairs)
                t_sort += time.perf_counter() - t0
                keys_done += n
                n_sorts += 1
                if pairs:
                    ok = np.array_equal(gk.cpu().numpy(), exp[0]) and \
                        np.array_equal(gv.cpu().numpy().view(np.uint32), exp[1].view(np.uint32))
                else:
                    g = gk.cpu().numpy()
                    ok = np.array_equal(g.view(np.uint8), np.ascontiguousarray(exp).view(np.uint8))
                check["checked"] += 1
                check["failed"] += 0 if ok else 1
        finally:
            unpin(old)
        for (o, idx, (gk, gv)) in to_check[n_sorts:]:  # beyond the oracle budget: properties
            check["checked"] += 1
            inp = pristine[(o, idx % ninst)]
            check["failed"] += 0 if check_props(gk, inp, gv, vals_pristine if pairs else None) else 1
        check["how"] = (f"{n_sorts} outputs bit-exact vs the oracle, "
                        f"{len(to_check) - n_sorts} by properties (sorted, multiset fingerprints"
                        + (", payload invariants" if pairs else "") + ")")
        cpu = {"value": round(keys_done / t_sort / 1e6, 3), "unit": "Mkeys/s", "cores": 1, "kind": "oracle",
               "sample": f"{n_sorts} of the {len(to_check)} timed instances of {orders} (n={n}), "
                         "single-threaded C mergesort" + (f" pinned to core {core}" if core is not None else ""),
               "host_cpus": os.cpu_count()}
    else:
        for (o, idx, (gk, gv)) in to_check:
            check["checked"] += 1
            inp = pristine[(o, idx % ninst)]
            check["failed"] += 0 if check_props(gk, inp, gv, vals_pristine if pairs else None) else 1
        check["how"] = "properties on the device (sorted, multiset fingerprints" + (
            ", payload invariants" if pairs else "") + ")"
    if big and not big_same:
        check["failed"] += 1
    del kept, first_big, to_check

    # ---- the flushed variant (rotate runs only): restore + 512 MiB write before every sort, which
    # also evicts the kernels' code; a few steps, same events, for comparison
    flushed = None
    if rotate:
        fsteps = min(steps, 5)
        clk_f = ClockSampler(dev.index).__enter__()
        for o in orders:
            one_sort(o, 0, flushed=True)
        fev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in orders]
               for _ in range(fsteps)]
        for s in range(fsteps):
            for j, o in enumerate(orders):
                one_sort(o, warm + s, fev[s][j], flushed=True)
        torch.cuda.synchronize()
        clk_f.__exit__()
        clk.absorb(clk_f)
        fms = {o: statistics.mean(fev[s][j][0].elapsed_time(fev[s][j][1]) for s in range(fsteps))
               for j, o in enumerate(orders)}
        ftot = max_over_ranks(sum(fms.values()), dev)
        flushed = {"value": round(n * len(orders) * ws / (ftot / 1e3) / 1e6, 2), "unit": "Mkeys/s", "steps": fsteps,
                   "ms_per_step": round(ftot, 4), "per_order_ms_mean": {o: round(v, 4) for o, v in fms.items()},
                   "l2": L2_TEXT["flush"]}

    # ---- e2e through the host API (pinned host buffers, copies inside the events)
    e2e = None
    if not args.no_e2e:
        clk_e = ClockSampler(dev.index).__enter__()
        pin = {o: torch.from_numpy(host_inputs[(o, 0)]).pin_memory() for o in orders}
        hbuf = torch.empty(shape, dtype=tdt).pin_memory()
        hb = hbuf.numpy()
        hv = None
        if pairs:
            hvals = torch.empty(n, dtype=torch.int32).pin_memory()
            hv = hvals.numpy()
            hvals_src = torch.from_numpy(gen.index_payload(n).view(np.int32)).pin_memory()
        e2e_ms = 0.0
        for s in range(warm + steps):
            for o in orders:
                hbuf.copy_(pin[o])
                if pairs:
                    hvals.copy_(hvals_src)
                flush.fill_(s)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if rec:  # records have no host-buffer entry point: H2D, sort, D2H through torch + sr
                    work.copy_(hbuf, non_blocking=True)
                    sr.sort_records(work)
                    hbuf.copy_(work, non_blocking=True)
                else:
                    sr.sort_host(hb, hv, stream.cuda_stream)
                b.record(stream)
                b.synchronize()
                if s >= warm:
                    e2e_ms += a.elapsed_time(b)
        e2e_ms = max_over_ranks(e2e_ms, dev)
        e2e = {"value": round(keys_all / (e2e_ms / 1e3) / 1e6, 2), "unit": "Mkeys/s",
               "h2d_bytes_per_step": n * kw * len(orders), "d2h_bytes_per_step": n * kw * len(orders),
               "ms_per_step": round(e2e_ms / steps, 4), "call": "sr_sort_host, one call per instance"}
        if not rec and len(orders) > 1:
            # the step's instances as ONE sr_sort_host_batch call: uploads, sorts and downloads of
            # neighbouring instances overlap (same bytes, same pinned buffers, every output checked)
            hbufs = [torch.empty(shape, dtype=tdt).pin_memory() for _ in orders]
            hvs = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in orders] if pairs else None
            bat_ms, bad = 0.0, 0
            for s in range(warm + steps):
                for hbo, o in zip(hbufs, orders):
                    hbo.copy_(pin[o])
                for hvo in hvs or []:
                    hvo.copy_(hvals_src)
                flush.fill_(s)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sr.sort_host_batch([h.numpy() for h in hbufs], [h.numpy() for h in hvs] if pairs else None,
                                   stream.cuda_stream)
                b.record(stream)
                b.synchronize()
                if s >= warm:
                    bat_ms += a.elapsed_time(b)
                if s == warm + steps - 1:  # the last step's outputs against the serial path's (verified above)
                    for hbo, o in zip(hbufs, orders):
                        hbuf.copy_(pin[o])
                        if pairs:
                            hvals.copy_(hvals_src)
                        sr.sort_host(hb, hv, stream.cuda_stream)
                        ibits = np.int32 if hbo.element_size() == 4 else np.int64  # (bit patterns: NaN keys)
                        bad += 0 if np.array_equal(hbo.numpy().view(ibits), hbuf.numpy().view(ibits)) else 1
                        if not hbo.is_floating_point():
                            hk_np = hbo.numpy()
                            bad += 0 if bool(np.all(hk_np[:-1] <= hk_np[1:])) else 1
                    for hvo in hvs or []:
                        bad += 0 if torch.equal(hvo, hvals) else 1
            bat_ms = max_over_ranks(bat_ms, dev)
            if bad:
                raise SystemExit(f"bench: {bad} batched e2e outputs differ from sr_sort_host's or are unsorted")
            e2e = {"value": round(keys_all / (bat_ms / 1e3) / 1e6, 2), "unit": "Mkeys/s",
                   "h2d_bytes_per_step": e2e["h2d_bytes_per_step"], "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                   "ms_per_step": round(bat_ms / steps, 4),
                   "call": "sr_sort_host_batch, the step's instances in one call (copies overlap the sorts)",
                   "per_call": {"value": e2e["value"], "ms_per_step": e2e["ms_per_step"], "call": e2e["call"]}}
            del hbufs, hvs
        clk_e.__exit__()
        clk.absorb(clk_e)
        del pin, hbuf

    # ---- per-kernel device times (profile pass over the same inputs, CUDA events on the sort stream)
    sr.set_option(sr.OPT_PROFILE, 1)
    kern = {}
    if rotate:
        restore_all()
    for s in range(steps):
        for o in orders:
            one_sort(o, warm + s)
            for name, ms, by in sr.last_profile():
                d = kern.setdefault(name, {"ms": 0.0, "bytes": 0, "launches": 0})
                d["ms"] += ms
                d["bytes"] += by
                d["launches"] += 1
    sr.set_option(sr.OPT_PROFILE, 0)
    hbm, hbm_src = peaks()
    dname, d = max(kern.items(), key=lambda kv: kv[1]["ms"])
    avg_ms = d["ms"] / d["launches"]
    bytes_per_launch = d["bytes"] / d["launches"]
    achieved = bytes_per_launch / (avg_ms / 1e3) / 1e9
    kern_total = sum(v["ms"] for v in kern.values())
    tr = ncu_traffic(dname, "int" if elem_bytes(dtype) == 4 else "long", wl)
    roofline = {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": tr["bytes"] if tr else None,
                "traffic_source": tr, "algorithmic_bytes_per_launch": int(bytes_per_launch),
                "avg_launch_ms": round(avg_ms, 5), "peak_source": hbm_src,
                "share_of_kernel_time": round(d["ms"] / kern_total, 3),
                "kernels": {k: {"ms_per_launch": round(v["ms"] / v["launches"], 4),
                                "GBps": round(v["bytes"] / v["launches"] / (v["ms"] / v["launches"] / 1e3) / 1e9, 1),
                                "launches_per_step": v["launches"] / steps} for k, v in kern.items()}}
    step_ms_mean = total_ms / steps
    del pristine, work, flush, works, works_v
    torch.cuda.empty_cache()
    return {
        "value": round(value, 2), "ms_per_step": round(step_ms_mean, 4), "dtype": dtype_label(dtype) + (
            "+u32 payload" if pairs else ""),
        "detail": {"per_order_ms_mean": {o: round(statistics.mean(v), 4) for o, v in per_order_ms.items()},
                   "total_of_order_means_ms": round(sum(statistics.mean(v) for v in per_order_ms.values()), 4),
                   "routes": route_of, "wall_s": round(t_wall, 3), "l2_mode": "rotate" if rotate else "flush",
                   **({"l2_flushed": flushed} if flushed else {}),
                   "parallelism": f"independent instances per rank x{ws}"},
        "whole_step_hbm": {"bytes_planned_per_step": int(bytes_planned),
                           "GBps": round(bytes_planned / (step_ms_mean / 1e3) / 1e9, 1),
                           "frac_of_peak": round(bytes_planned / (step_ms_mean / 1e3) / 1e9 / hbm, 4),
                           "ideal_pass_frac": round(2 * n * kw * len(orders) / (step_ms_mean / 1e3) / 1e9 / hbm, 4)},
        "roofline": roofline, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e,
        "verified": check, "cpu_baseline": cpu,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="c2", choices=list(WORKLOADS))
    ap.add_argument("--sub", default="c5a", help="second workload reported inside the same line ('none' to skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--l2", default="rotate", choices=["rotate", "flush"],
                    help="keep inputs out of L2 by rotating input buffers (when the run's inputs are >= 4 L2 "
                         "sizes) or by a 512 MiB write before every sort (see l2_mode)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = args.workload

    if args.impl == "reference":
        run_reference(args, wl)
        return

    import torch
    import paper_1609_04471_b200 as sr

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    oracle_leg = rank == 0 and ws == 1 and not args.no_cpu_baseline

    m = measure(wl, args, sr, dev, stream, rank, ws, oracle_leg)
    sub = None
    if args.sub and args.sub != "none" and args.sub != wl:
        sm = measure(args.sub, args, sr, dev, stream, rank, ws, oracle_leg)
        sub = {"workload": args.sub, "config": ref_config(args.sub, args), "value": sm["value"], "unit": "Mkeys/s",
               "ms_per_step": sm["ms_per_step"], "dtype": sm["dtype"], **{k: sm[k] for k in (
                   "detail", "whole_step_hbm", "roofline", "gpu_launches", "clocks", "e2e", "verified",
                   "cpu_baseline")}}
    failed = m["verified"]["failed"] + (sub["verified"]["failed"] if sub else 0)
    line = {
        "metric": METRIC, "value": m["value"], "unit": "Mkeys/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": m["dtype"], "data": "synthetic", "config": ref_config(wl, args),
        "detail": m["detail"], "whole_step_hbm": m["whole_step_hbm"], "roofline": m["roofline"],
        "gpu_launches": m["gpu_launches"], "clocks": m["clocks"], "verified": m["verified"],
    }
    if m["e2e"]:
        line["e2e"] = m["e2e"]
    if m["cpu_baseline"]:
        line["cpu_baseline"] = m["cpu_baseline"]
    if sub:
        line[args.sub] = sub
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    if failed:
        print(f"bench: {failed} sorted outputs failed verification", file=sys.stderr, flush=True)
        sys.exit(3)


if __name__ == "__main__":
    main()
