#!/usr/bin/env python
"""Benchmark of the B200 RNS-CKKS hot path (BASELINE.json metric):
HMult+relin and HRot throughput at N=2^16 (l=24, alpha=8, dnum=3).

One step = one batch of B independent ciphertexts per GPU:
    B x HMult+relinearize (merged ModDown+rescale, l=24 -> 22) and
    B x HRot(r=1) (ModUp / KeyMult / ModDown / automorphism, l=24),
inputs resident in HBM (`value`), and the same through the public API with
the step's ciphertexts copied host->device from pinned memory and the results
copied back (`e2e`).  Data-parallel over ranks (weak scaling, no collective in
the step): `python -m torch.distributed.run --nproc-per-node N bench.py --gpus N`.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, built read-only from /root/reference) on the same metric.
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
from fractions import Fraction
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# enough hardware work queues that concurrently spinning peer-exchange waits of
# virtual limb shards (one stream each) never queue behind each other
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

N_RING, L, ALPHA, DB, LEVEL = 1 << 16, 24, 8, 55, 24
METRIC = "HMult+relin & HRot ops/s at N=2^16 (l=24, alpha=8, dnum=3)"
UNIT = "ops/s"
LIMB = N_RING * 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=48, help="ciphertexts per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=3, help="concurrent sub-batches (CUDA streams) per GPU")
    ap.add_argument("--split", choices=["batch", "ops"], default="batch",
                    help="2-stream schedule: 'batch' = each stream runs HMult then HRot on half the batch; 'ops' = "
                         "one stream runs HMult, the other HRot, each on the whole batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=4, help="ciphertexts per H2D/compute/D2H chunk")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the B=1 eager / CUDA-graph measurement")
    ap.add_argument("--no-sweep", action="store_true", help="skip the HRot level x batch sweep (config 2)")
    ap.add_argument("--workload", default="dp", choices=["dp", "limb", "helr"],
                    help="dp: batched independent ciphertexts (configs 1-3, the headline); limb: one ciphertext "
                         "limb-sharded over the ranks at N=2^17 (config 4); helr: HELR-style logistic-regression "
                         "iteration (config 5)")
    ap.add_argument("--exchange", choices=["gather", "peer"], default="peer",
                    help="config 4 exchange: NCCL all-gather + copy, or peer-mapped loads inside BConv "
                         "(CUDA IPC across ranks; default)")
    ap.add_argument("--no-graph", action="store_true", help="helr: skip the CUDA-graph replay measurement")
    ap.add_argument("--no-extra", action="store_true",
                    help="default line: skip the config 4 (limb, N=2^17) and config 5 (HELR) sub-measurements")
    ap.add_argument("--virtual-shards", type=int, default=0,
                    help="limb workload on ONE GPU: drive this many shards from one process (exchange = local "
                         "copies); measures the summed shard compute, not multi-GPU speed")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) is polled every 2 ms from a thread — an nvidia-smi
    process takes ~100 ms per query, longer than a default timed region —
    with one nvidia-smi query as the fallback when NVML is unavailable."""

    # nvmlClocksEventReason* bits (nvml.h)
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.bits = [], [], 0
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
            while True:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.bits |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self._ready.set()
                if self._stop.wait(0.002):
                    break
            nv.nvmlShutdown()
            return
        except Exception:
            pass
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,"
                                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            self._ready.set()
            r = [x.strip() for x in out.stdout.strip().split(",")]
            self.sm.append(float(r[0]))
            self.mx.append(float(r[1]))
            for bit, v in zip((0x8, 0x40, 0x20, 0x4), r[2:6]):
                if v.lower() == "active":
                    self.bits |= bit
        except Exception:
            pass

    def __enter__(self):
        # NVML initialises before the timed region starts: wait for the first sample
        self._ready = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=5)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(v for k, v in self.REASONS.items() if self.bits & k), "samples": len(self.sm)}


def dist_setup():
    """(world, rank, local device index) for this process; initialises the
    process group (NCCL; CK32_DIST_BACKEND=gloo exercises the N > 1 code path
    with several ranks sharing the GPUs of a smaller box, LOCAL_RANK modulo
    the device count)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    numa_local(local)  # also at N = 1: the e2e leg's pinned buffers are first-touched on the GPU's NUMA node
    if world > 1:
        backend = os.environ.get("CK32_DIST_BACKEND", "nccl")
        t0 = time.perf_counter()
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        # force the communicator into existence now (NCCL creates it lazily)
        # and say so, so a launcher can match ranks to GPUs
        probe = torch.ones(1, device=torch.device("cuda", local) if backend == "nccl" else "cpu")
        dist.all_reduce(probe)
        print(f"[bench] rank {rank}/{world}: {backend} communicator up on cuda:{local} "
              f"({torch.cuda.get_device_name(local)}, all-reduce check {int(probe.item())} == {world}) "
              f"in {time.perf_counter() - t0:.2f} s", file=sys.stderr, flush=True)
    return world, rank, local


def numa_local(device: int) -> None:
    """Pin this rank's host threads to the CPUs NVML reports as local to its
    GPU, so the pinned e2e buffers (first-touch) and the launch thread live on
    the GPU's NUMA node.  Best effort: no NVML, no change."""
    try:
        import pynvml as nv

        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(device)
        words = nv.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            print(f"[bench] cuda:{device}: host threads pinned to {len(cpus)} NUMA-local CPUs", file=sys.stderr)
        nv.nvmlShutdown()
    except Exception:
        pass


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------- CPU legs --
def cpu_reference_times(reps: int, warmup: int, ndebug: bool = False):
    """The reference's own mechanism benchmark (bench.cpp:332-389), all host
    cores; ndebug=True runs the same sources built with -DNDEBUG (SURVEY
    §8(d): the shipped build keeps asserts live, proj/CMakeLists.txt:10)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from pyoracle import Reference

    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    ref = Reference(ndebug=ndebug)
    hm = ref.mechanism_bench("hmult", N_RING, L, ALPHA, DB, LEVEL, reps, warmup)
    hr = ref.mechanism_bench("hrot", N_RING, L, ALPHA, DB, LEVEL, reps, warmup)
    return hm, hr


def cpu_baseline_leg():
    """Both CPU columns of SURVEY §8(d); `value` is the faster (-DNDEBUG)
    build so the GPU/CPU ratio is taken against the strongest legal baseline."""
    out = {}
    for key, nd in (("as_shipped", False), ("ndebug", True)):
        try:
            hm, hr = cpu_reference_times(reps=5, warmup=1, ndebug=nd)
            per_pair = (hm["median_ns"] + hr["median_ns"]) * 1e-9
            out[key] = {"value": round(2.0 / per_pair, 4), "cores": hm["omp_threads"],
                        "hmult_ms": round(hm["median_ns"] / 1e6, 2), "hrot_ms": round(hr["median_ns"] / 1e6, 2),
                        "build": "reference sources -O3 " + ("-DNDEBUG" if nd else "as shipped (asserts live)")
                                 + ", Boost shim"}
        except Exception as e:  # reference build (oracle/_ref) missing
            out[key] = {"value": None, "error": f"{type(e).__name__}: {e}"}
    best = out["ndebug"] if out["ndebug"].get("value") else out["as_shipped"]
    if not best.get("value"):
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": best.get("error")}
    return {"value": best["value"], "unit": UNIT, "cores": best["cores"], "kind": "reference",
            "sample": "reference bench::run_mechanism_bench hmult + hrot(r=1) at N=2^16 l=24 alpha=8, "
                      "median of 5 reps each (1 ciphertext at a time, OpenMP inside the op)",
            "build": best["build"], "hmult_ms": best["hmult_ms"], "hrot_ms": best["hrot_ms"],
            "columns": out}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warm = max(args.steps, 1), max(args.warmup, 0)
    # the -DNDEBUG build of the reference's own sources (the faster legal
    # baseline); the as-shipped build when that one is not built
    try:
        hm, hr = cpu_reference_times(reps=steps, warmup=warm, ndebug=True)
        build = "reference sources -O3 -DNDEBUG, Boost shim"
    except FileNotFoundError:
        hm, hr = cpu_reference_times(reps=steps, warmup=warm)
        build = "reference sources -O3 as shipped (asserts live), Boost shim"
    per_pair = (hm["median_ns"] + hr["median_ns"]) * 1e-9
    v = 2.0 / per_pair
    line = {"metric": METRIC, "value": round(v, 4), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": round(per_pair * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32 residues (u32 mod q < 2^29, int64 accum)",
            "data": "synthetic (reference keygen/encrypt of random unit-disk slots, seed 42)",
            "config": {"workload": "1 HMult+relin + 1 HRot(r=1) per step at N=2^16, l=24, alpha=8, dnum=3 "
                                   "(reference CPU path, one ciphertext at a time)", "n": N_RING, "l": L,
                       "alpha": ALPHA, "level": LEVEL},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": hm["omp_threads"], "kind": "reference",
                             "sample": f"median of {steps} reps of hmult and of hrot via bench::run_mechanism_bench",
                             "build": build},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "hmult_ms": round(hm["median_ns"] / 1e6, 2), "hrot_ms": round(hr["median_ns"] / 1e6, 2)}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- GPU leg ----
def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.workload == "limb":
        run_limb(args)
        return
    if args.workload == "helr":
        run_helr(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_13055_b200 import ckks, dp
    from paper_2407_13055_b200.pipeline import HostPipeline

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()

    B = args.batch
    C = ckks.CkksContext(ckks.CkksParams(n=N_RING, l=L, alpha=ALPHA, delta_bits=DB), device=local)
    q = torch.tensor(C.primes.astype(np.int64), device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def rand_rows(shape_prefix, rows_q):  # uniform residues per row (synthetic)
        u = torch.randint(0, 1 << 62, (*shape_prefix, len(rows_q), N_RING), device=dev, generator=gen,
                          dtype=torch.int64)
        return (u % q[rows_q].view(*([1] * len(shape_prefix)), -1, 1)).to(torch.int32).contiguous()

    qrows = torch.arange(LEVEL, device=dev)
    full = torch.cat([torch.arange(L, device=dev), L + torch.arange(ALPHA, device=dev)])
    D = C.num_digits(L)
    relin = ckks.EvaluationKey(rand_rows((D, 2), full), ckks.RELIN)
    rot = ckks.EvaluationKey(rand_rows((D, 2), full), ckks.ROTATION, 1)
    s = Fraction(1 << DB)
    X = ckks.Ciphertext(rand_rows((B, 2), qrows), s, LEVEL)
    Y = ckks.Ciphertext(rand_rows((B, 2), qrows), s, LEVEL)
    st = torch.cuda.current_stream(dev)

    def step():
        o1 = ckks.hmult(C, X, Y, relin)
        o2 = ckks.hrot(C, X, 1, rot)
        return o1, o2

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)

    # concurrent sub-batches: the batch is split over `streams` CUDA streams
    # (each with its own scratch arena) so one sub-batch's memory-bound
    # kernels overlap another's integer-bound ones.
    S_n = max(1, min(args.streams, B))
    subs = [dp.shard_bounds(B, S_n, i) for i in range(S_n)]
    streams = [st] + [torch.cuda.Stream(dev) for _ in range(S_n - 1)]

    def concurrent_step():
        start = torch.cuda.Event()
        start.record(st)
        done, outs = [], []
        if args.split == "ops" and S_n == 2:  # HMult on one stream, HRot on the other, whole batch each
            res = []
            for k, s_k in enumerate(streams):
                s_k.wait_event(start)
                with torch.cuda.stream(s_k):
                    res.append(ckks.hmult(C, X, Y, relin).data if k == 0 else ckks.hrot(C, X, 1, rot).data)
                    e = torch.cuda.Event()
                    e.record(s_k)
                    done.append(e)
            for e in done:
                st.wait_event(e)
            return [(res[0], res[1])]
        for (lo, hi), s_k in zip(subs, streams):
            s_k.wait_event(start)
            with torch.cuda.stream(s_k):
                Xs = ckks.Ciphertext(X.data[lo:hi], s, LEVEL)
                Ys = ckks.Ciphertext(Y.data[lo:hi], s, LEVEL)
                outs.append((ckks.hmult(C, Xs, Ys, relin).data, ckks.hrot(C, Xs, 1, rot).data))
                e = torch.cuda.Event()
                e.record(s_k)
                done.append(e)
        for e in done:
            st.wait_event(e)
        return outs  # read only after a device synchronize

    if S_n > 1:
        for _ in range(2):
            concurrent_step()
        torch.cuda.synchronize(dev)

    # ---- main timed region: inputs resident in HBM (B x 25 MB >> 126 MB L2)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * args.steps)]
    l0 = C.launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(st)
        for k in range(args.steps):
            if S_n > 1:
                concurrent_step()
                continue
            ev[3 * k].record(st)
            ckks.hmult(C, X, Y, relin)
            ev[3 * k + 1].record(st)
            ckks.hrot(C, X, 1, rot)
            ev[3 * k + 2].record(st)
        t_end.record(st)
        torch.cuda.synchronize(dev)
    barrier()
    launches = C.launch_count() - l0
    ms = t_start.elapsed_time(t_end)
    if S_n > 1:  # per-op rates from a short sequential pass (not part of `value`)
        for k in range(args.steps):
            ev[3 * k].record(st)
            ckks.hmult(C, X, Y, relin)
            ev[3 * k + 1].record(st)
            ckks.hrot(C, X, 1, rot)
            ev[3 * k + 2].record(st)
        torch.cuda.synchronize(dev)
    hm_ms = sum(ev[3 * k].elapsed_time(ev[3 * k + 1]) for k in range(args.steps))
    hr_ms = sum(ev[3 * k + 1].elapsed_time(ev[3 * k + 2]) for k in range(args.steps))
    ms_max, hm_ms, hr_ms = dp.max_over_ranks([ms, hm_ms, hr_ms], device=dev)  # device time, max over ranks
    ops_total = 2 * B * args.steps * world
    value = ops_total / (ms_max / 1e3)

    # ---- correctness of the configuration just timed: one more step in the
    # timed schedule (B split over S_n streams with per-stream scratch arenas),
    # then the first and last ciphertext of every sub-batch recomputed alone
    # (B = 1, default stream; that path is pinned to the reference's full-size
    # hashes by tests/test_gpu_parity.py) and compared residue for residue.
    outs = concurrent_step() if S_n > 1 else [step()]
    outs = [(o1.data, o2.data) if hasattr(o1, "data") else (o1, o2) for o1, o2 in outs]
    torch.cuda.synchronize(dev)
    checked, bit_exact = [], True
    for (lo, hi), (o1, o2) in zip(subs if (S_n > 1 and args.split == "batch") else [(0, B)], outs):
        for b in sorted({lo, hi - 1}):
            X1 = ckks.Ciphertext(X.data[b:b + 1].contiguous(), s, LEVEL)
            Y1 = ckks.Ciphertext(Y.data[b:b + 1].contiguous(), s, LEVEL)
            r1 = ckks.hmult(C, X1, Y1, relin).data
            r2 = ckks.hrot(C, X1, 1, rot).data
            ok = bool(torch.equal(r1[0], o1[b - lo])) and bool(torch.equal(r2[0], o2[b - lo]))
            bit_exact &= ok
            checked.append(b)
    del outs
    bit_exact = bool(dp.max_over_ranks([0.0 if bit_exact else 1.0], device=dev)[0] == 0.0)

    # ---- per-kernel-class breakdown (CUDA events around every launch group)
    C.profile(True)
    for _ in range(max(1, min(args.steps, 3))):
        step()
    prof = C.profile_read()
    C.profile(False)
    hbm, peak_kind = peaks()
    tot_ms = sum(p["ms"] for p in prof) or 1.0
    dom = max(prof, key=lambda p: p["ms"])
    ntt = next(p for p in prof if p["name"] == "ntt_fwd")
    kern = []
    for p in prof:
        if p["groups"]:
            kern.append({"kernel": p["name"], "share": round(p["ms"] / tot_ms, 4),
                         "GBps": round(p["bytes"] / (p["ms"] * 1e6), 1),
                         "frac": round(p["bytes"] / (p["ms"] * 1e6) / hbm, 4)})

    try:
        traffic_ratio = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
    except Exception:
        traffic_ratio = {}

    def roof(p):
        ach = p["bytes"] / (p["ms"] * 1e6)
        per_group = p["bytes"] / max(p["groups"], 1)
        tr = traffic_ratio.get(p["name"], {}).get("ratio")
        return {"kernel": p["name"], "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": round(tr * per_group) if tr else None,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full DRAM bytes per algorithmic byte)"
                if tr else None, "peak_kind": peak_kind,
                "bytes_per_launch_group": round(p["bytes"] / max(p["groups"], 1)),
                "avg_group_ms": round(p["ms"] / max(p["groups"], 1), 4),
                "timing": "CUDA events around every launch group on its launching stream (ck_profile), over "
                          "steps of the same workload run on one stream right after the timed region: in the "
                          "2-stream timed region the two streams' kernels overlap, so per-kernel spans there "
                          "would count the other stream's time"}

    def int_pipe(p):
        """INT-pipe view of an NTT class (report it beside GB/s).
        A radix-2 N=2^16 limb is 16 x 32768 butterflies for 524,288 algorithmic
        bytes, so butterflies/s == algorithmic B/s."""
        bfly_s = p["bytes"] / (p["ms"] * 1e-3)
        mhz = clk.summary().get("sm_mhz") or 1965.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        per = bfly_s / (sms * mhz * 1e6)
        return {"butterflies_per_clk_per_sm": round(per, 2), "ceiling": 11.7,
                "ceiling_source": "Shoup butterfly microbenchmark, tools/microbench_bfly2.cu "
                                  "(profiles/round1_session2.md)", "frac": round(per / 11.7, 3)}

    # ---- e2e: host ciphertexts in pinned memory, H2D + compute + D2H every step
    e2e = None
    if not args.no_e2e:
        Be = B
        hx = torch.empty((Be, 2, LEVEL, N_RING), dtype=torch.int32).pin_memory()
        hy = torch.empty_like(hx).pin_memory()
        hx.copy_(X.data[:Be].cpu())
        hy.copy_(Y.data[:Be].cpu())
        ho1 = torch.empty((Be, 2, LEVEL - 2, N_RING), dtype=torch.int32).pin_memory()
        ho2 = torch.empty((Be, 2, LEVEL, N_RING), dtype=torch.int32).pin_memory()
        pipe = HostPipeline(dev, chunk=max(1, min(args.e2e_chunk, Be)), depth=2)

        def e2e_fn(d, o):  # results written into the pipeline's per-slot buffers (no allocation per step)
            cx = ckks.Ciphertext(d[0], s, LEVEL)
            o1 = ckks.hmult(C, cx, ckks.Ciphertext(d[1], s, LEVEL), relin, out=o[0])
            o2 = ckks.hrot(C, cx, 1, rot, out=o[1])
            return o1.data, o2.data

        def e2e_step():  # the whole batch: H2D, HMult + HRot, D2H (chunked, overlapped)
            return pipe.run([hx, hy], e2e_fn, [ho1, ho2], outputs_in_place=True)

        for _ in range(max(args.warmup, 1)):  # warm the pinned buffers' DMA mappings too
            e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.steps):
            last = e2e_step()
        st.wait_event(last)
        b.record(st)
        torch.cuda.synchronize(dev)
        e_ms = dp.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        e2e = {"value": round(2 * Be * args.steps * world / (e_ms / 1e3), 2), "unit": UNIT,
               "h2d_bytes_per_step": int(hx.numel() * 4 * 2), "d2h_bytes_per_step": int((ho1.numel() + ho2.numel()) * 4),
               "path": "ckks.hmult / ckks.hrot (C ABI) on ciphertexts copied from pinned host memory; results copied "
                       "back each step (pipeline.HostPipeline: chunks of %d, H2D / compute / D2H on separate "
                       "streams, results written into per-slot device buffers: no allocation per step)" % pipe.chunk}
        # the link's own ceiling for this step: the same H2D and D2H bytes copied concurrently
        # (two streams, nothing else running), best of 3 -- e2e / ceiling says how close the
        # pipeline gets to PCIe, the bound of the end-to-end number
        din = [torch.empty_like(hx, device=dev), torch.empty_like(hy, device=dev)]
        dout = [torch.empty_like(ho1, device=dev), torch.empty_like(ho2, device=dev)]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        best = None
        for _ in range(3):
            torch.cuda.synchronize(dev)
            a.record(st)
            s_in.wait_event(a)
            s_out.wait_event(a)
            with torch.cuda.stream(s_in):
                for d_, h_ in zip(din, (hx, hy)):
                    d_.copy_(h_, non_blocking=True)
            with torch.cuda.stream(s_out):
                for h_, d_ in zip((ho1, ho2), dout):
                    h_.copy_(d_, non_blocking=True)
            st.wait_stream(s_in)
            st.wait_stream(s_out)
            b.record(st)
            torch.cuda.synchronize(dev)
            best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
        ceil_ops = 2 * Be / (best / 1e3)
        e2e["pcie_ceiling"] = {"copy_only_ms_per_step": round(best, 3),
                               "bidirectional_GBps": round((e2e["h2d_bytes_per_step"] + e2e["d2h_bytes_per_step"]) / (best * 1e6), 1),
                               "ops_per_s": round(ceil_ops, 1), "frac": round(e2e["value"] / world / ceil_ops, 3)}
        del din, dout

    # ---- single-ciphertext serving (B = 1): eager C-ABI calls vs one CUDA graph replay
    small = None
    if not args.no_small:
        from paper_2407_13055_b200.pipeline import CapturedStep

        X1 = ckks.Ciphertext(X.data[:1].contiguous(), s, LEVEL)
        Y1 = ckks.Ciphertext(Y.data[:1].contiguous(), s, LEVEL)

        def one():
            return ckks.hmult(C, X1, Y1, relin).data, ckks.hrot(C, X1, 1, rot).data

        reps = 50
        for _ in range(3):
            one()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            one()
        b.record(st)
        torch.cuda.synchronize(dev)
        eager_ms = a.elapsed_time(b) / reps
        cap = CapturedStep(dev, one)
        a.record(st)
        for _ in range(reps):
            cap.replay()
        b.record(st)
        torch.cuda.synchronize(dev)
        graph_ms = a.elapsed_time(b) / reps
        s2 = torch.cuda.Stream(dev)

        def one_forked():  # HMult and HRot on two streams inside the same graph
            cur = torch.cuda.current_stream(dev)
            s2.wait_stream(cur)
            m = ckks.hmult(C, X1, Y1, relin).data
            with torch.cuda.stream(s2):
                r = ckks.hrot(C, X1, 1, rot).data
            cur.wait_stream(s2)
            return m, r

        cap2 = CapturedStep(dev, one_forked)
        a.record(st)
        for _ in range(reps):
            cap2.replay()
        b.record(st)
        torch.cuda.synchronize(dev)
        graph2_ms = a.elapsed_time(b) / reps
        small = {"batch": 1, "eager_ops_per_s": round(2 / (eager_ms / 1e3), 1),
                 "cuda_graph_ops_per_s": round(2 / (graph_ms / 1e3), 1),
                 "cuda_graph_2_streams_ops_per_s": round(2 / (graph2_ms / 1e3), 1),
                 "note": "one HMult+relin + one HRot per step on one ciphertext; graph = pipeline.CapturedStep "
                         "(2 streams: HMult and HRot forked inside the graph)"}

    # ---- config 2: HRot over every level (batch B) and a batch sweep at four levels
    sweep = grid = None
    if not args.no_sweep:
        Xbig = X.data.repeat(-(-128 // B), 1, 1, 1)[:max(128, B)] if B < 128 else X.data  # up to B = 128

        def hrot_rate(Bs, lv, reps=3):
            Xl = ckks.Ciphertext(Xbig[:Bs, :, :lv].contiguous(), s, lv)
            ckks.hrot(C, Xl, 1, rot)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(reps):
                ckks.hrot(C, Xl, 1, rot)
            b.record(st)
            torch.cuda.synchronize(dev)
            return round(reps * Bs / (a.elapsed_time(b) / 1e3), 1)

        sweep = {lv: hrot_rate(B, lv) for lv in range(LEVEL, 0, -2)}
        grid = {f"l{lv}": {f"B{bs}": hrot_rate(bs, lv) for bs in (1, 2, 4, 8, 16, 32, 64, 128) if bs <= Xbig.shape[0]}
                for lv in range(LEVEL, 0, -2)}
        del Xbig

    # ---- BASELINE configs 4 and 5 on this GPU, so the driver-run line carries
    # them: the N=2^17 single-ciphertext workload unsharded and as 8 virtual
    # limb shards (peer-memory exchange between the shards' buffers), and one
    # HELR iteration eager and replayed as a CUDA graph.  (Multi-GPU runs of
    # these use --workload limb / helr under torchrun.)
    extra = {}
    if world == 1 and not args.no_extra:
        import copy

        extra["config1_ntt_roundtrip"] = ntt_roundtrip(C, dev, st, clk)
        C.close()
        torch.cuda.empty_cache()
        c4 = {}
        for g in (0, 8):
            a4 = copy.copy(args)
            a4.virtual_shards, a4.exchange = g, "peer"
            d = limb_measure(a4, 1, 0, local)
            c4["unsharded" if g == 0 else f"virtual_shards_{g}"] = {
                "ops_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                "graph_ms_per_step": d["graph_ms_per_step"], "graph_ops_per_s": d["graph_ops_per_s"],
                "bit_exact_vs_single_device": d["bit_exact_vs_single_device"], "gpu_launches": d["gpu_launches"]}
            torch.cuda.empty_cache()
        extra["config4_limb_n131072"] = dict(
            c4, workload="BASELINE config 4: 1 HMult+relin + 1 HRot(r=1) per step on ONE ciphertext at N=2^17, "
                         "l=24, alpha=8; virtual shards = the limb-sharded path driven on one GPU (shard-local "
                         "kernels + peer-memory BConv exchange), i.e. summed shard compute, not multi-GPU speed")
        a5 = copy.copy(args)
        a5.no_graph = False
        d = helr_measure(a5, 1, 0, local)
        extra["config5_helr"] = {"it_per_s": d["value"], "ms_per_iteration": d["ms_per_iteration"],
                                 "eager_ms_per_iteration": d["eager_ms_per_iteration"],
                                 "graph_ms_per_iteration": d["graph_ms_per_iteration"],
                                 "gpu_launches": d["gpu_launches"], "workload": d["config"]["workload"]}

    if rank == 0:
        cpu = None if args.no_cpu or world > 1 else cpu_baseline_leg()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int32 residues (u32 mod q < 2^29, int64 accum)",
            "data": "synthetic uniform residues (ciphertexts and keys), random-init",
            "config": {"workload": f"per GPU per step: {B} x HMult+relin (merged rescale, l=24->22) + {B} x HRot(r=1) "
                                   f"at N=2^16, l=24, alpha=8, dnum=3 (configs[1]/[2] of BASELINE.json)",
                       "n": N_RING, "l": L, "alpha": ALPHA, "level": LEVEL, "batch_per_gpu": B,
                       "parallelism": f"dp{world} (independent ciphertexts, no collective)", "streams_per_gpu": S_n,
                       "stream_split": args.split,
                       "l2": "inputs larger than L2 (2 x B x 12 MiB ciphertext pairs per step); keys stay L2-resident"},
            "hmult_ops_per_s": round(B * args.steps * world / (hm_ms / 1e3), 2),
            "hrot_ops_per_s": round(B * args.steps * world / (hr_ms / 1e3), 2),
            "roofline": roof(dom),
            "roofline_ntt": dict(roof(ntt), int_pipe=int_pipe(ntt)),
            "kernels": kern,
            "gpu_launches": int(launches),
            "bit_exact": bit_exact,
            "bit_exact_check": f"one extra step of the timed schedule ({S_n} streams, per-stream arenas); ciphertexts "
                               f"{checked} of the batch recomputed alone (B=1) and compared residue for residue "
                               f"(HMult and HRot outputs); the B=1 path is pinned to the reference's full-size "
                               f"hashes in tests/test_gpu_parity.py",
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        line.update(extra)
        if small:
            line["single_ciphertext"] = small
        if sweep:
            line["hrot_level_sweep_ops_per_s"] = sweep
            line["hrot_level_batch_sweep_ops_per_s"] = grid
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ntt_roundtrip(C, dev, st, clk, rows: int = 3072, reps: int = 5):
    """BASELINE config 1's NTT/INTT round trip through the C ABI
    (ck_ntt_forward / ck_intt_inverse, ntt.hpp:90-91): `rows` limbs of
    N = 2^16 cycling over the 32 primes (3072 x 256 KiB = 768 MiB, larger
    than L2), forward then inverse, each timed with CUDA events on the
    library's (current) stream over `reps` repetitions; the round trip must
    return the input residues exactly."""
    import numpy as np
    import torch
    from paper_2407_13055_b200 import _native as nat

    g = np.array([i % (L + ALPHA) for i in range(rows)], np.uint32)
    q = torch.tensor(C.primes[g].astype(np.int64), device=dev)
    x0 = (torch.randint(0, 1 << 62, (rows, N_RING), device=dev, dtype=torch.int64) % q[:, None]).to(torch.int32)
    x = x0.clone()
    garr = nat.u32_array(g)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fwd = lambda: nat.call("ck_ntt_forward", C.handle, x.data_ptr(), rows, garr, C.stream())  # noqa: E731
    inv = lambda: nat.call("ck_intt_inverse", C.handle, x.data_ptr(), rows, garr, None, C.stream())  # noqa: E731
    fwd()
    inv()
    exact = bool(torch.equal(x, x0))
    out = {}
    peak, kind = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clk.summary().get("sm_mhz") or 1965.0
    # reps forward transforms, then reps inverse ones: the inverse is exact on
    # canonical residues, so x ends where it started
    for name, fn in (("fwd", fwd), ("inv", inv)):
        torch.cuda.synchronize(dev)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / reps
        gbs = rows * 8 * N_RING / (ms * 1e6)
        bfly = rows * 16 * (N_RING // 2) / (ms * 1e-3) / (sms * mhz * 1e6)
        out[name] = {"ms": round(ms, 4), "ns_per_limb": round(ms * 1e6 / rows, 1), "GBps": round(gbs, 1),
                     "frac": round(gbs / peak, 4), "butterflies_per_clk_per_sm": round(bfly, 2)}
    exact = exact and bool(torch.equal(x, x0))
    del x, x0
    torch.cuda.empty_cache()
    return dict(out, roundtrip_exact=exact, limbs=rows, peak_GBps=peak, peak_kind=kind,
                bytes_per_limb=8 * N_RING,
                workload="BASELINE config 1 NTT/INTT round trip: %d limbs of N=2^16 over the 32 primes "
                         "(768 MiB, larger than L2), C ABI ck_ntt_forward / ck_intt_inverse, %d reps each" % (rows, reps))


def run_limb(args):
    """Config 4: one ciphertext, RNS limbs sharded over the ranks (N=2^17,
    l=24, alpha=8); one step = 1 HMult+relin (merged rescale) + 1 HRot(r=1),
    each with two all-gathers (ModUp sources, ModDown sources) over NCCL."""
    import torch.distributed as dist

    world, rank, local = dist_setup()
    line = limb_measure(args, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def limb_measure(args, world, rank, local, graph=True):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_13055_b200 import ckks, dp
    from paper_2407_13055_b200.limb import (MERGED, MOD_DOWN, IpcPeerExchange, LimbShardedEvaluator, LocalExchange,
                                            LocalPeerExchange, ShardBackend, TorchExchange, exchange_bytes)

    n = 1 << 17
    dev = torch.device("cuda", local)
    C = ckks.CkksContext(ckks.CkksParams(n=n, l=L, alpha=ALPHA, delta_bits=DB), device=local)
    q = torch.tensor(C.primes.astype(np.int64), device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321)  # same synthetic ciphertext and keys on every rank

    def rand_rows(prefix, rows):
        u = torch.randint(0, 1 << 62, (*prefix, len(rows), n), device=dev, generator=gen, dtype=torch.int64)
        return (u % q[rows].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()

    full = torch.cat([torch.arange(L, device=dev), L + torch.arange(ALPHA, device=dev)])
    qrows = torch.arange(LEVEL, device=dev)
    D = C.num_digits(L)
    relin, rotk = rand_rows((D, 2), full), rand_rows((D, 2), full)
    x, y = rand_rows((2,), qrows), rand_rows((2,), qrows)
    if args.virtual_shards and world == 1:
        G = args.virtual_shards
        shards = [ShardBackend(C, G, r) for r in range(G)]
        exch = LocalPeerExchange(shards) if args.exchange == "peer" else LocalExchange()
    else:
        G = world
        shards = [ShardBackend(C, world, rank)]
        if args.exchange == "peer":
            exch = IpcPeerExchange(shards[0]) if world > 1 else LocalPeerExchange(shards)
        else:
            exch = TorchExchange() if world > 1 else LocalExchange()
    lays = [s.layout for s in shards]
    # virtual shards run side by side on their own streams, as they would on separate GPUs
    ev = LimbShardedEvaluator(shards, exch, concurrent=bool(args.virtual_shards and world == 1))
    xs = [lay.split_ct(x, LEVEL) for lay in lays]
    ys = [lay.split_ct(y, LEVEL) for lay in lays]
    rk = [lay.split_key(relin) for lay in lays]
    ok = [lay.split_key(rotk) for lay in lays]
    del relin, rotk
    st = torch.cuda.current_stream(dev)

    def step():
        ev.hmult(LEVEL, xs, ys, rk)
        ev.hrot(LEVEL, xs, 1, ok)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    l0 = C.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.steps):
            step()
        b.record(st)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = dp.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
    launches = C.launch_count() - l0
    # The whole step replayed as one CUDA graph per rank, which removes the
    # host launch cost of the ~30 small kernels per mechanism and shard: the
    # peer exchange keeps its epochs and buffer parities in device memory, so
    # a captured step replays across processes too.
    graph_ms = None
    if graph and (world == 1 or args.exchange == "peer"):
        from paper_2407_13055_b200.pipeline import CapturedStep
        cap = CapturedStep(dev, step)
        for _ in range(max(args.warmup, 1)):
            cap.replay()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        a.record(st)
        for _ in range(args.steps):
            cap.replay()
        b.record(st)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        graph_ms = dp.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        del cap
    # correctness spot check against the single-device path (rank-local rows)
    if world == 1:
        X = ckks.Ciphertext(x, Fraction(1 << DB), LEVEL)
        Y = ckks.Ciphertext(y, Fraction(1 << DB), LEVEL)
        full_hm = ckks.hmult(C, X, Y, ckks.EvaluationKey(_unsplit(rk, lays)))
        got = torch.cat(ev.hmult(LEVEL, xs, ys, rk), dim=1)
        exact = bool(torch.equal(got, full_hm.data))
    else:
        exact = None
    peer_errors = exch.errors() if hasattr(exch, "errors") else None
    if peer_errors and any(peer_errors):
        raise RuntimeError(f"peer exchange timed out: {peer_errors}")
    line = None
    if rank == 0:
        xb = exchange_bytes(lays[0], n, LEVEL, MERGED) + exchange_bytes(lays[0], n, LEVEL, MOD_DOWN)
        line = {
            "metric": "single-ciphertext limb-sharded HMult+relin & HRot ops/s at N=2^17 (l=24, alpha=8, dnum=3)",
            "value": round(2 * args.steps / (ms / 1e3), 2), "unit": "ops/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32 residues (u32 mod q < 2^29, int64 accum)",
            "data": "synthetic uniform residues (ciphertext and keys), random-init",
            "config": {"workload": "BASELINE config 4: 1 HMult+relin (merged rescale) + 1 HRot(r=1) per step on one "
                                   "ciphertext at N=2^17, l=24, alpha=8, limbs sharded over the ranks; BConv source "
                                   "rows exchanged before ModUp and ModDown: "
                                   + ("peer-mapped loads inside BConv (CUDA IPC, epoch flags)" if args.exchange == "peer"
                                      else "NCCL all-gather + copy"),
                       "exchange": args.exchange,
                       "n": n, "l": L, "alpha": ALPHA, "level": LEVEL, "shards": G,
                       "virtual_shards_on_one_gpu": bool(args.virtual_shards and world == 1),
                       "parallelism": f"limb-sharded x{G}"},
            "exchange_bytes_received_per_rank_per_step": xb,
            "graph_ms_per_step": round(graph_ms / args.steps, 4) if graph_ms else None,
            "graph_ops_per_s": round(2 * args.steps / (graph_ms / 1e3), 2) if graph_ms else None,
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "bit_exact_vs_single_device": exact,
        }
    if world > 1:
        dist.barrier()  # no rank frees its exchange buffer while a peer may still read it
    if hasattr(exch, "close"):
        exch.close()
    for sh in shards:
        sh.close()
    C.close()
    return line


def run_helr(args):
    """Config 5: HELR-style logistic-regression iteration (helr.py) at N=2^16,
    l=24, one mini-batch of 8 ciphertexts x (128 samples x 256 features) per
    GPU (1024 samples, the batch of Cheddar's HELR run).
    Synthetic ciphertexts, keys and plaintext constants (uniform residues)."""
    import torch.distributed as dist

    world, rank, local = dist_setup()
    line = helr_measure(args, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def helr_measure(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_13055_b200 import ckks, dp
    from paper_2407_13055_b200.helr import HelrIteration, HelrShape

    dev = torch.device("cuda", local)
    shape = HelrShape(n=N_RING, features=256, cts=8)
    C = ckks.CkksContext(ckks.CkksParams(n=N_RING, l=L, alpha=ALPHA, delta_bits=DB), device=local)
    q = torch.tensor(C.primes.astype(np.int64), device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(777 + rank)

    def rand_rows(prefix, rows):
        u = torch.randint(0, 1 << 62, (*prefix, len(rows), N_RING), device=dev, generator=gen, dtype=torch.int64)
        return (u % q[rows].view(*([1] * len(prefix)), -1, 1)).to(torch.int32).contiguous()

    full = torch.cat([torch.arange(L, device=dev), L + torch.arange(ALPHA, device=dev)])
    D = C.num_digits(L)
    relin = ckks.EvaluationKey(rand_rows((D, 2), full))
    keys = {r: ckks.EvaluationKey(rand_rows((D, 2), full), ckks.ROTATION, r) for r in shape.rotations()}

    def const(level, scale):
        return ckks.Plaintext(ckks.Polynomial(rand_rows((), torch.arange(level, device=dev)), level, 0), scale, level)

    it = HelrIteration(C, shape, relin, keys, {k: const for k in ("mask", "a3", "a1", "a0", "gamma", "one")})
    s = Fraction(1 << DB)
    Z = ckks.Ciphertext(rand_rows((shape.cts, 2), torch.arange(L, device=dev)), s, L)
    W = ckks.Ciphertext(rand_rows((2,), torch.arange(L, device=dev)), s, L)
    st = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 0)):
        it.step(Z, W)
    torch.cuda.synchronize(dev)
    l0 = C.launch_count()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.steps):
            it.step(Z, W)
        b.record(st)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = dp.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
    eager_ms = ms
    graph_ms = None
    if not args.no_graph:  # the same iteration captured once in a CUDA graph and replayed (pipeline.CapturedStep)
        from paper_2407_13055_b200.pipeline import CapturedStep
        cap = CapturedStep(dev, lambda: it.step(Z, W))
        for _ in range(max(args.warmup, 1)):
            cap.replay()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a.record(st)
        for _ in range(args.steps):
            cap.replay()
        b.record(st)
        torch.cuda.synchronize(dev)
        graph_ms = dp.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        ms = min(ms, graph_ms)
    line = None
    if rank == 0:
        per = ms / args.steps
        line = {
            "metric": "HELR-style logistic-regression iterations/s (1024-sample mini-batch per GPU, N=2^16, l=24)",
            "value": round(world * args.steps / (ms / 1e3), 2), "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per, 4), "ms_per_iteration": round(per, 4),
            "eager_ms_per_iteration": round(eager_ms / args.steps, 4),
            "graph_ms_per_iteration": round(graph_ms / args.steps, 4) if graph_ms else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32 residues (u32 mod q < 2^29, int64 accum)",
            "data": "synthetic uniform residues (ciphertexts, keys, plaintext constants), random-init",
            "config": {"workload": "BASELINE config 5: one HELR gradient step (helr.py): 8 ciphertexts x 128 "
                                   "samples x 256 features, inner products by rotate-and-sum, mask + replicate, "
                                   "degree-3 sigmoid, gradient sum over samples, batched mechanisms", "n": N_RING, "l": L, "alpha": ALPHA,
                       "features": shape.features, "samples": shape.cts * shape.samples_per_ct,
                       "rns_limbs_consumed": it.levels_used(), "ops_per_iteration": it.op_profile(),
                       "parallelism": f"dp{world} (one mini-batch per GPU)"},
            "gpu_launches": int(C.launch_count() - l0), "clocks": clk.summary(),
        }
    C.close()
    return line


def _unsplit(keys, lays):
    """reassemble shard-local keys [D][2][q+p] into the full [D][2][L+alpha] key"""
    import torch
    qs = [k[:, :, :lay.q_hi - lay.q_lo] for k, lay in zip(keys, lays)]
    ps = [k[:, :, lay.q_hi - lay.q_lo:] for k, lay in zip(keys, lays)]
    return torch.cat(qs + ps, dim=2).contiguous()


if __name__ == "__main__":
    main()
