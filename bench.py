#!/usr/bin/env python
"""Benchmark: nonlocal stiffness assembly on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Default workload: C4 (BASELINE configs[4]: N=96, delta=3h, fullcaps M=128,
7.0e9 element pairs), the largest configuration that fits one B200 and the
one the multi-GPU scaling is quoted on.  One "step" = one full assembly (nlfem::assemble analogue: element pairs ->
pattern -> FP64 integration -> CSR) of the named workload.  Prints ONE JSON
line (rank 0).

  value      element-pair integrals/s, device-timed (CUDA events on the
             launching stream) with the element table resident in HBM
  e2e        same metric through the C-ABI one-shot call nlfem_gpu_assemble
             with host arrays: H2D upload + device pipeline + CSR D2H per step
  roofline   the integration kernel (k_integrate, FP64-pipe bound) against the
             FP64 DFMA peak measured live by nlfem_gpu_fp64_peak()
  cpu_baseline  the unmodified reference assemble() (oracle/_ref, all host
             cores) on a bounded sample of the workload (see sample_cfg)

--impl reference times the unmodified reference's assemble() (oracle/_ref,
its own mesh generator and element table; nothing from paper_2302_07499_b200
is imported) on this box's host cores, one reference assemble() of the
sample mesh per step (rank 0 only), and prints the same line with
"impl": "reference" and the same `config`.

--gpus N without torchrun re-launches itself under torch.distributed.run.

Multi-GPU (torchrun, NCCL): owner-computes -- each rank builds the pairs of a
contiguous range of outer elements, its local node pattern and their exact
fixed-point partial sums, ships the slots of other ranks' rows to their owners
(all-to-all of the halo records), finalizes its own row block from what it
received (bit-identical to one GPU) and the row blocks are all-gathered on
device (paper_2302_07499_b200/distributed.py).  Total work is fixed: scaling
"strong".
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
    # C3f without the jitter and C4 with it (overlap-mode diagnostics: size or structure?)
    "P48s": dict(res=48, delta=3 / 48, strategy="fullcaps", mc=128, jitter=None),
    "P96j": dict(res=96, delta=3 / 96, strategy="fullcaps", mc=128, jitter=7),
}
METRIC = "element-pair integrals/s"
# B200 FP64 (non-tensor) nominal: 148 SMs x 64 DFMA/clk x 2 FLOP x 1.965 GHz
FP64_NOMINAL_TF = 148 * 64 * 2 * 1.965e9 / 1e12

# dram__bytes_read.sum + dram__bytes_write.sum of the units kernels (all k_mc
# launches of one step, or of one chunk scaled to the step) from the committed
# ncu --set full captures; None where no capture was taken for that workload
TRAFFIC = {"C1": (432594432, "profiles/r1_c1_kmc_ncu.txt (dram read+write summed over the "
                             "step's k_mc launches)"),
           # one units chunk's 8 k_mc launches: 2,208,101,632 B for 8,388,608 element
           # pairs (~264 B per pair, mostly the 80-B item records), times the step's
           # 7,012,417,536 pairs
           "C4": (1846e9, "profiles/r3d_c4_kmc_ncu.txt (dram read+write of one chunk's k_mc "
                          "launches, ncu --set full, scaled by element pairs to the step)")}


def describe(name, cfg):
    d = dict(cfg)
    s = (f"{name}: structured N={cfg['res']} cubes/side (6 tets each) + layer, "
         f"delta={cfg['delta']:.6g}, {cfg['strategy']}")
    if cfg["strategy"] == "fullcaps":
        s += f", M={cfg['mc']} per MC sub-simplex, Philox4x32-7 seed {SEED}"
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


# The reference's per-element-pair rate at fixed delta/h and M does not depend
# on the mesh size (same Monte Carlo draws per pair, 760.8 at delta = 3h,
# M = 128, for every N; measured rates N = 8 / 12 / 16 / 24 in
# profiles/r2_ref_rate_vs_n.txt), so the reference's CPU time is sampled on
# the N = SAMPLE_RES mesh at the workload's delta/h and M: one step of the
# reference arm is one full reference assemble() of that mesh (seconds of CPU
# work), where the benchmarked C2-C4 workloads would take hours.
SAMPLE_RES = 8


def sample_cfg(cfg):
    """The bounded CPU sample of a workload (same delta/h, strategy, M)."""
    if cfg["res"] <= 12:
        return dict(cfg), "full workload"
    ratio = cfg["delta"] * cfg["res"]
    s = dict(cfg, res=SAMPLE_RES, delta=ratio / SAMPLE_RES)
    note = (f"[est.] N={SAMPLE_RES} mesh at the workload's delta/h={ratio:g} and M: the "
            "per-element-pair rate is mesh-size independent at fixed delta/h "
            "(profiles/r2_ref_rate_vs_n.txt)")
    return s, note


def reference_sample(cfg):
    """The unmodified reference (oracle/_ref) on the sample mesh: its own
    generate_mesh / build_cmap / build_element_table / build_dofmap, plus the
    element pairs of the sample counted by the restated oracle on the
    reference's own table.  Imports nothing from paper_2302_07499_b200."""
    import types
    from oracle import port, ref
    s, note = sample_cfg(cfg)
    coords, cells, region = ref.generate_mesh(s["res"], s["delta"], jitter_seed=s["jitter"])
    R = ref.Problem(coords, cells, region)
    t = types.SimpleNamespace(**R.table())
    t.coords = np.ascontiguousarray(coords, np.float64)
    t.elem_count, t.node_count, t.unknowns = R.elems, R.nodes, R.unknowns
    Cc, f = ref.forcing(s["delta"], U2)
    # the pair set does not depend on M (mode R: the reference's own stream)
    o = port.assemble(t, s["delta"], s["strategy"], Cc, f, U2, seed=SEED, mc_samples=1,
                      sampler="R", threads=os.cpu_count() or 1)
    sample = (f"{s['strategy']} N={s['res']} delta={s['delta']:.6g} M={s['mc']}: {note}; "
              f"unmodified reference assemble(), AssemblyStats.seconds")
    return R, s, int(o["element_pairs"]), sample


def reference_steps(R, s, steps, cores):
    out = []
    for _ in range(steps):
        r = R.assemble(s["delta"], s["strategy"], U2, threads=cores, seed=SEED,
                       mc_samples=s["mc"])
        out.append(r["seconds"])
    return out


def cpu_baseline(cfg):
    """One bounded reference run beside the GPU line (rank 0, N=1)."""
    cores = os.cpu_count() or 1
    R, s, pairs, sample = reference_sample(cfg)
    t = reference_steps(R, s, 1, cores)
    return {"value": pairs / t[0], "unit": "element-pair integrals/s", "cores": cores,
            "kind": "reference", "sample": sample}


def run_reference_arm(args, cfg_name, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    R, s, pairs, sample = reference_sample(cfg)
    reference_steps(R, s, max(args.warmup, 0), cores)
    times = reference_steps(R, s, args.steps, cores)
    tot = sum(times)
    value = pairs * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": METRIC,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfg_name, cfg),
        "parallelism": f"reference assemble() on {cores} host threads (rank 0)",
        "sample_element_pairs": pairs,
        "cpu_baseline": {"value": value, "unit": METRIC, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_JSON_OUT, flush=True)
    return 0


def bench_config(cfg_name, cfg):
    """The `config` object: identical in both arms (the workload, nothing else)."""
    return {"workload": describe(cfg_name, cfg)["text"], "name": cfg_name}


_JSON_OUT = sys.stdout


def self_launch(args) -> int | None:
    """`--gpus N` without a torchrun environment: re-launch this command as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1
    rendezvous); the rank-0 JSON line reaches this process's stdout."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return None
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def system_sha(sess, dist_out=None) -> str:
    """SHA-256 of the assembled system (row offsets, columns, values, rhs as
    raw bytes): the bitwise check of N-GPU runs against one GPU."""
    import hashlib
    import torch
    ro, ci, va, rh = (torch.as_tensor(x, device="cuda") for x in sess.outputs())
    if dist_out is not None:
        va, ci, rh, ro = dist_out
    h = hashlib.sha256()
    for t in (ro, ci, va, rh):
        h.update(t.contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--verify", action="store_true",
                    help="add the SHA-256 of the assembled system to the line")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU (sharded, NCCL) path even on one rank: exercises "
                         "the N>1 code on a single GPU")
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        return rc
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
            return D.device_step(sess, stream=stream.cuda_stream)
    else:
        def step():
            return None, sess.run(stream.cuda_stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    launches_per_step = sess.launches()

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    step_ms, k3_ms, mc_ms = [], [], []
    st = out = None
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 between timed steps (inputs are smaller than L2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out, st = step()
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
    sha = system_sha(sess, out) if args.verify else None
    stats = {"element_pairs": int(st.element_pairs), "items": int(st.items),
             "mc_samples": int(st.mc_samples), "mc_hits": int(st.mc_hits)}
    ledger, ledger_units = int(st.ledger_flops), int(st.ledger_flops_units)
    k3 = float(np.mean(k3_ms))
    kmc = float(np.mean(mc_ms))
    if dist is not None:  # each rank counts its own outer elements: sum over ranks
        c = torch.tensor([*stats.values(), ledger, ledger_units], dtype=torch.int64,
                         device="cuda")
        dist.all_reduce(c)
        c = [int(x) for x in c.cpu()]
        stats = dict(zip(stats, c[:4]))
        ledger, ledger_units = c[4], c[5]
        tk = torch.tensor([k3, kmc], dtype=torch.float64, device="cuda")
        dist.all_reduce(tk, op=dist.ReduceOp.MAX)  # the slowest rank's phases
        k3, kmc = (float(x) for x in tk.cpu())
    pairs = stats["element_pairs"]
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
        res = None
        nwarm = 1  # the first call also sets up the workspace and the pinned result pool
        nsteps = max(1, min(args.steps, 3))
        ws = None
        for i in range(nsteps + nwarm):
            res = None  # release the previous result (its pinned block goes back to the pool)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            if not use_dist:
                res, _ = P.assemble(table, cfg["delta"], cfg["strategy"], "moment2", U2,
                                    seed=SEED, mc_samples=cfg["mc"], device=local)
            else:  # upload into the rank's workspace session (reused, like the one-shot
                # call's), sharded assembly, row blocks gathered to host on every rank
                if ws is None:
                    ws = P.Session(table, cfg["delta"], cfg["strategy"], "moment2", U2,
                                   seed=SEED, mc_samples=cfg["mc"], device=local)
                else:
                    ws.reset(table)
                res, _ = D.assemble_distributed(ws)
            t1 = time.perf_counter()
            dt = t1 - t0
            if dist is not None:
                tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if i >= nwarm:
                e2e_t.append(dt)
            d2h = sum(res[k].nbytes for k in ("row_ptr", "col_idx", "values", "rhs"))
        if ws is not None:
            ws.close()
        e2e = {"value": pairs / float(np.mean(e2e_t)), "unit": METRIC,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * float(np.mean(e2e_t)), "steps": len(e2e_t),
               "path": "nlfem_gpu_assemble (one-shot C-ABI call, host arrays)" if not use_dist
               else "assemble_distributed (sharded, host CSR on every rank)"}

    peak = P.fp64_peak_tflops(local)
    # dominant kernel: the units kernels (k_mc: inner pieces + Monte Carlo; its
    # launches run on two streams, timed together by CUDA events around them).
    # N > 1: the ledger of all ranks over the slowest rank's phase time, per GPU
    units = kmc > 0 and ledger_units > 0
    if units:
        achieved = ledger_units / (kmc * 1e-3) / 1e12 / world
        rl_kernel, rl_flops, rl_ms = ("k_mc (units phase: inner pieces + Monte Carlo, all "
                                      "launches of one step)"), ledger_units, kmc
    else:  # barycenter / overlap / inside: whole-element items in the combine only
        achieved = ledger / (k3 * 1e-3) / 1e12 / world
        rl_kernel, rl_flops, rl_ms = "k_integrate (combine)", ledger, k3
    integ = ledger / (k3 * 1e-3) / 1e12 / world
    traffic = TRAFFIC.get(args.config) if units and world == 1 else None
    # overlap mode: multi-chunk Monte Carlo runs time the units
    # phase while it shares each SM with the previous chunk's combine
    overlap_on = (cfg["strategy"] == "fullcaps" and pairs / world > 2 * (1 << 23)
                  and os.environ.get("NLFEM_COMB_OVERLAP", "3") not in ("0", "2"))
    overlap_note = ("on: the units phase shares each SM with the previous chunk's combine, which "
                    "runs as one resident CTA per SM (k_mc alone, NLFEM_COMB_OVERLAP=0: 0.555 of "
                    "the measured peak at C4, profiles/r3b_overlap_mode.txt)") if overlap_on else "off"
    line = {
        "metric": METRIC, "value": value, "unit": METRIC,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, cfg),
        "parallelism": (f"outer-element shards x{world} "
                        f"({os.environ.get('NLFEM_BENCH_BACKEND', 'nccl').upper()} "
                        "owner-computes: halo records all-to-all + row-block all-gather)")
        if use_dist else "single GPU",
        "l2": "flushed between steps (256 MiB write; inputs smaller than L2)",
        **stats,
        "fp64_gflops_ledger": ledger / (t_total / args.steps * 1e-3) / 1e9,
        "phase_ms": [round(x, 3) for x in st.phase_ms[:6]],
        "roofline": {"kernel": rl_kernel, "bound": "fp64", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": "of measured: nlfem_gpu_fp64_peak() DFMA microbenchmark, "
                                    "this run (burst); MEASURED_PEAKS.json has no FP64 figure",
                     "peak_nominal": FP64_NOMINAL_TF,
                     "frac_of_nominal": achieved / FP64_NOMINAL_TF,
                     "ledger_flops_per_launch": int(rl_flops), "launch_ms": rl_ms,
                     "overlap": overlap_note,
                     "traffic": traffic[0] if traffic else None,
                     "traffic_source": traffic[1] if traffic else None,
                     "integration_phase": {"kernels": "k_mc + k_integrate", "ms": k3,
                                           "ledger_flops": int(ledger),
                                           "achieved": integ, "frac": integ / peak}},
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk,
    }
    if sha:
        line["system_sha256"] = sha
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as exc:  # report, never fail the bench line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
