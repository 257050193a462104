#!/usr/bin/env python
"""Benchmark: nonlocal stiffness assembly on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl ours|reference]

One "step" = one full assembly (nlfem::assemble analogue: element pairs ->
pattern -> FP64 integration -> CSR) of the named workload.  Prints ONE JSON
line (rank 0).

  value      element-pair integrals/s, device-timed (CUDA events on the
             launching stream) with the element table resident in HBM
  e2e        same metric through the C-ABI one-shot call nlfem_gpu_assemble
             with host arrays: H2D upload + device pipeline + CSR D2H per step
  roofline   the integration kernel (k_integrate, FP64-pipe bound) against the
             FP64 DFMA peak measured live by nlfem_gpu_fp64_peak()
  cpu_baseline  the unmodified reference assemble() (oracle/_ref, all host
             cores) on the same workload, when built; else the CPU port

--impl reference times the reference's own CPU assemble() on this box's host
cores for the same config (rank 0 only) and prints the same line with
"impl": "reference".

Multi-GPU (torchrun, NCCL): the assembly is sharded -- each rank integrates a
contiguous range of outer elements into exact fixed-point partial sums, an
int64 all-reduce combines them (bit-identical to one GPU), each rank finalizes
its row block and the row blocks are all-gathered on device
(paper_2302_07499_b200/distributed.py).  Total work is fixed: scaling "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

U2 = np.array([[1, 2, 0, 0], [1, 0, 2, 0], [1, 0, 0, 2]], float)  # u = |x|^2, f = -6
SEED = 1234

# BASELINE.json configs; mc_samples per Monte Carlo sub-simplex (reference semantics)
CONFIGS = {
    "C0": dict(res=8, delta=0.25, strategy="barycenter", mc=1, jitter=None),
    "C1": dict(res=8, delta=0.25, strategy="fullcaps", mc=64, jitter=None),
    "C2": dict(res=32, delta=0.1, strategy="fullcaps", mc=256, jitter=None),
    "C3n": dict(res=48, delta=3 / 48, strategy="nocaps", mc=1, jitter=7),
    "C3f": dict(res=48, delta=3 / 48, strategy="fullcaps", mc=128, jitter=7),
    "C4": dict(res=96, delta=3 / 96, strategy="fullcaps", mc=128, jitter=None),
    # the other strategies on the config-1 mesh (not BASELINE workloads)
    "C1n": dict(res=8, delta=0.25, strategy="nocaps", mc=1, jitter=None),
    "C1a": dict(res=8, delta=0.25, strategy="approxcaps", mc=1, jitter=None),
    # smaller same-delta/h variants for profiling
    "P3n": dict(res=24, delta=3 / 24, strategy="nocaps", mc=1, jitter=7),
    "P3f": dict(res=24, delta=3 / 24, strategy="fullcaps", mc=128, jitter=7),
}
# B200 FP64 (non-tensor) nominal: 148 SMs x 64 DFMA/clk x 2 FLOP x 1.965 GHz
FP64_NOMINAL_TF = 148 * 64 * 2 * 1.965e9 / 1e12

# dram__bytes_read.sum + dram__bytes_write.sum of the units kernels (all k_mc
# launches of one step) from the committed ncu --set full capture; None where
# no capture was taken for that workload
TRAFFIC = {"C1": 432594432}


def describe(name, cfg):
    d = dict(cfg)
    s = (f"{name}: structured N={cfg['res']} cubes/side (6 tets each) + layer, "
         f"delta={cfg['delta']:.6g}, {cfg['strategy']}")
    if cfg["strategy"] == "fullcaps":
        s += f", M={cfg['mc']} per MC sub-simplex, Philox4x32-10 seed {SEED}"
    if cfg["jitter"] is not None:
        s += f", interior vertices jittered +-0.2h (seed {cfg['jitter']})"
    s += ", moment2 kernel (gamma=15/(2 pi delta^5)), u=|x|^2, f=-6, FP64"
    d["text"] = s
    return d


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.source = "nvidia-smi, every 0.2 s"
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        """NVML handle of this process's CUDA device (matched by PCI bus id)."""
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:  # in-process NVML, sampled every 5 ms (short timed regions)
            nv, h = self._nvml_handle()
            names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown",
                     0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def nvml_loop():
                while not self._stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        act = ["Active" if bits & b else "Not Active" for b in names]
                        self.rows.append([str(self.index), str(sm), str(mx), "", hex(bits),
                                          act[0], act[1], act[2], act[3]])
                    except Exception:
                        pass
                    self._stop.wait(0.005)
            self._t = threading.Thread(target=nvml_loop, daemon=True)
            self._t.start()
            self.source = "nvml, every 5 ms"
            return
        except Exception:
            pass

        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    for line in out.strip().splitlines():
                        self.rows.append([x.strip() for x in line.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows), "sampler": self.source}


def cpu_baseline(cfg_name, cfg, steps=1):
    """Reference assemble() on this host's cores; bounded sample of the workload."""
    from oracle import ref, port
    import paper_2302_07499_b200 as P
    sample = dict(cfg)
    note = "full workload"
    if cfg["res"] > 12:
        # same delta/h and M on a smaller mesh; pairs/s is per-outer-element work
        ratio = cfg["delta"] * cfg["res"]
        sample["res"] = 10 if cfg["strategy"] != "fullcaps" else 8
        sample["delta"] = ratio / sample["res"]
        note = (f"N={sample['res']} mesh at the same delta/h={ratio:g} and M; rate per element "
                "pair is mesh-size independent at fixed delta/h")
    m = P.generate_mesh(3, sample["res"], sample["delta"], jitter_seed=sample["jitter"])
    cores = os.cpu_count() or 1
    times, pairs = [], None
    if ref.available():
        R = ref.Problem(m["coords"], m["cells"], m["region"])
        for _ in range(steps):
            out = R.assemble(sample["delta"], sample["strategy"], U2, threads=cores, seed=SEED,
                             mc_samples=sample["mc"])
            times.append(out["seconds"])
        kind = "reference"
    else:
        t = P.ElementTable(m["coords"], m["cells"], m["region"])
        for _ in range(steps):
            t0 = time.perf_counter()
            port.assemble(t, sample["delta"], sample["strategy"],
                          P.kernel_constant(sample["delta"], "moment2"),
                          P.forcing_terms(sample["delta"], U2, "moment2"), P.normalize_terms(U2),
                          seed=SEED, mc_samples=sample["mc"], sampler="R", threads=cores)
            times.append(time.perf_counter() - t0)
        kind = "port"
    # element pairs of the sample (count with the GPU pair kernel when available)
    pairs = count_pairs(m, sample)
    return dict(times=times, pairs=pairs, cores=cores, kind=kind, note=note,
                sample=f"{sample['strategy']} N={sample['res']} delta={sample['delta']:.6g} "
                       f"M={sample['mc']}: {note}")


def count_pairs(m, cfg):
    """Element pairs (T,T') with a piece for some quad point of T (the metric's
    unit), counted by the restated CPU oracle outside any timed region, so the
    reference arm never touches the GPU code."""
    from oracle import port
    import paper_2302_07499_b200 as P
    t = P.ElementTable(m["coords"], m["cells"], m["region"])
    mc = 1 if cfg["strategy"] != "fullcaps" else 1  # pair sets do not depend on M
    o = port.assemble(t, cfg["delta"], cfg["strategy"], P.kernel_constant(cfg["delta"], "moment2"),
                      P.forcing_terms(cfg["delta"], U2, "moment2"), P.normalize_terms(U2),
                      seed=SEED, mc_samples=mc, sampler="P", threads=os.cpu_count() or 1)
    return int(o["element_pairs"])


def run_reference_arm(args, cfg_name, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_baseline(cfg_name, cfg, steps=1)
    cb = cpu_baseline(cfg_name, cfg, steps=args.steps)
    tot = sum(cb["times"])
    value = cb["pairs"] * len(cb["times"]) / tot
    line = {
        "impl": "reference", "metric": "element-pair integrals/s", "value": value,
        "unit": "element-pair integrals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(cb["times"]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": describe(cfg_name, cfg)["text"], "name": cfg_name,
                   "element_pairs": int(cb["pairs"]),
                   "parallelism": f"reference assemble() on {cb['cores']} host threads (rank 0)"},
        "cpu_baseline": {"value": value, "unit": "element-pair integrals/s", "cores": cb["cores"],
                         "kind": cb["kind"], "sample": cb["sample"]},
        "e2e": {"value": value, "unit": "element-pair integrals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_JSON_OUT, flush=True)
    return 0


_JSON_OUT = sys.stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C1", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU (sharded, NCCL) path even on one rank: exercises "
                         "the N>1 code on a single GPU")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    # stdout carries exactly one JSON line: anything else written to file
    # descriptor 1 (NCCL's version banner, library prints) goes to stderr
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference_arm(args, args.config, cfg)

    import torch
    import paper_2302_07499_b200 as P

    rank, world, local = dist_env()
    if os.environ.get("NLFEM_BENCH_BACKEND", "nccl") != "nccl":
        local %= max(torch.cuda.device_count(), 1)  # test mode: ranks may share a GPU
    torch.cuda.set_device(local)
    dist = None
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        backend = os.environ.get("NLFEM_BENCH_BACKEND", "nccl")  # gloo: tests on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def barrier():
        if dist is not None:
            dist.barrier()

    m = P.generate_mesh(3, cfg["res"], cfg["delta"], jitter_seed=cfg["jitter"])
    # upstream setup (cmap, element table, dof map) on this rank's GPU
    table = P.ElementTable(m["coords"], m["cells"], m["region"], device=local)
    sess = P.Session(table, cfg["delta"], cfg["strategy"], "moment2", U2, seed=SEED,
                     mc_samples=cfg["mc"], device=local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2

    if use_dist:
        from paper_2302_07499_b200 import distributed as D

        def step():
            return D.device_step(sess, stream=stream.cuda_stream)[1]
    else:
        def step():
            return sess.run(stream.cuda_stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    launches_per_step = sess.launches()

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    step_ms, k3_ms, mc_ms = [], [], []
    st = None
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 between timed steps (inputs are smaller than L2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        k3_ms.append(st.phase_ms[3])
        mc_ms.append(st.phase_ms[5])
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t_total = sum(step_ms)
    if dist is not None:
        t = torch.tensor([t_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    pairs = int(st.element_pairs)  # all element pairs of the workload (every rank builds them)
    value = pairs * args.steps / (t_total * 1e-3)

    # end to end: one-shot C-ABI call with host arrays (upload + run + download).
    # The device-resident session is released first: at C4 its buffers alone
    # take ~70 GB and the one-shot call keeps its own workspace.
    sess.close()
    del flush
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        h2d = table.nbytes() + 8 * 8 * (len(sess.fterms) + len(sess.uterms))
        e2e_t = []
        d2h = 0
        out = None
        nwarm = 2  # the first calls also set up the workspace and the pinned result pool
        ws = None
        for i in range(max(1, min(args.steps, 3)) + nwarm):
            out = None  # release the previous result (its pinned block goes back to the pool)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            if not use_dist:
                out, _ = P.assemble(table, cfg["delta"], cfg["strategy"], "moment2", U2,
                                    seed=SEED, mc_samples=cfg["mc"], device=local)
            else:  # upload into the rank's workspace session (reused, like the one-shot
                # call's), sharded assembly, row blocks gathered to host on every rank
                if ws is None:
                    ws = P.Session(table, cfg["delta"], cfg["strategy"], "moment2", U2,
                                   seed=SEED, mc_samples=cfg["mc"], device=local)
                else:
                    ws.reset(table)
                out, _ = D.assemble_distributed(ws)
            t1 = time.perf_counter()
            dt = t1 - t0
            if dist is not None:
                tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if i >= nwarm:
                e2e_t.append(dt)
            d2h = sum(out[k].nbytes for k in ("row_ptr", "col_idx", "values", "rhs"))
        if ws is not None:
            ws.close()
        e2e = {"value": pairs / float(np.mean(e2e_t)), "unit": "element-pair integrals/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * float(np.mean(e2e_t))}

    peak = P.fp64_peak_tflops(local)
    k3 = float(np.mean(k3_ms))
    kmc = float(np.mean(mc_ms))
    # dominant kernel: the units kernels (k_mc: inner pieces + Monte Carlo; its
    # launches run on two streams, timed together by CUDA events around them)
    units = kmc > 0 and st.ledger_flops_units > 0
    if units:
        achieved = st.ledger_flops_units / (kmc * 1e-3) / 1e12
        rl_kernel, rl_flops, rl_ms = ("k_mc (units phase: inner pieces + Monte Carlo, all "
                                      "launches of one step)"), st.ledger_flops_units, kmc
    else:  # barycenter / overlap / inside: whole-element items in the combine only
        achieved = st.ledger_flops / (k3 * 1e-3) / 1e12
        rl_kernel, rl_flops, rl_ms = "k_integrate (combine)", st.ledger_flops, k3
    integ = st.ledger_flops / (k3 * 1e-3) / 1e12
    line = {
        "metric": "element-pair integrals/s", "value": value, "unit": "element-pair integrals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(args.config, cfg)["text"], "name": args.config,
                   "element_pairs": pairs, "items": int(st.items),
                   "mc_samples": int(st.mc_samples), "mc_hits": int(st.mc_hits),
                   "l2": "flushed between steps (256 MiB write; inputs smaller than L2)",
                   "parallelism": (f"outer-element shards x{world} "
                                   f"({os.environ.get('NLFEM_BENCH_BACKEND', 'nccl').upper()} "
                                   "int64 all-reduce + row-block all-gather)")
                                  if use_dist else "single GPU"},
        "fp64_gflops_ledger": st.ledger_flops / (t_total / args.steps * 1e-3) / 1e9,
        "phase_ms": [round(x, 3) for x in st.phase_ms[:6]],
        "roofline": {"kernel": rl_kernel, "bound": "fp64", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": "of measured: nlfem_gpu_fp64_peak() DFMA microbenchmark, "
                                    "this run (burst); MEASURED_PEAKS.json has no FP64 figure",
                     "peak_nominal": FP64_NOMINAL_TF,
                     "frac_of_nominal": achieved / FP64_NOMINAL_TF,
                     "ledger_flops_per_launch": int(rl_flops), "launch_ms": rl_ms,
                     "traffic": TRAFFIC.get(args.config) if units else None,
                     "traffic_source": "profiles/r1_c1_kmc_ncu.txt (dram read+write summed over "
                                       "the step's k_mc launches)" if units else None,
                     "integration_phase": {"kernels": "k_mc + k_integrate", "ms": k3,
                                           "ledger_flops": int(st.ledger_flops),
                                           "achieved": integ, "frac": integ / peak}},
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.config, cfg, steps=1)
            v = cb["pairs"] / min(cb["times"])
            line["cpu_baseline"] = {"value": v, "unit": "element-pair integrals/s",
                                    "cores": cb["cores"], "kind": cb["kind"],
                                    "sample": cb["sample"]}
        except Exception as exc:  # report, never fail the bench line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    sess.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
