#!/usr/bin/env python
"""bench.py -- PBN trajectory throughput on B200 (BASELINE.json metric).

A "step" is one pass of the whole hot path over one
batch of synthetic input: pbn_simulate on config C4 (n=2000, 16384 chains,
5e4 burn-in + 5e4 recorded transitions per chain, fused indicator /
transition / batch (kappa=500) counters, packed indicator bits, totals).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C4] [--chains N] [--burn-in B] [--window S]

Under torchrun (N > 1) every rank runs the same per-GPU workload on its own
chain range (weak scaling, no data-path collective); the max over ranks of
the device-timed region is used.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import CONFIGS, config_model, config_predicate  # noqa: E402

METRIC = "PBN node-updates/sec and chain-steps/sec on 1 B200; fraction of int/smem roofline"
UNIT = "node-updates/s"
SM_COUNT_B200 = 148


def demand_per_node_update(model, geometric: bool = False) -> dict:
    """Algorithmic demand per node-update, SURVEY §8(d) (declared from the
    method and the one-word-per-node-update stream of reading Q3, not from the
    achieved SASS), averaged over the nodes:
      RNG     1/4 Philox4x32-10 = 5 IMAD.WIDE (FMA pipe) + 5 LOP3 (ALU)
      decide  1 compare against T_p + (ell-1) compares/selects ~ ell + 1;
              nodes of the generic (dense, NEXT-3) path: a binary search,
              3 ops per step, ceil(log2 ell) steps
      gather  2 per parent of the selected function (extract + insert)
      lookup  2 (+1 word select when the selected function has theta >= 6)
      commit  1
    smem: (theta_sel + 1)/32 wavefronts (one state word per selected parent
    and one metadata read, each serving the 32 chains of a bit-sliced word).
    Image bytes (nodes of the generic path, image read through L1/L2): per
    lane the binary search's thresholds (4 B per step), the selected
    function's descriptor (16 B), its parent offsets (4 B each) and one
    table word (4 B); the node record (16 B) is shared by the 32 lanes.
    theta_sel, [theta >= 6] are weighted by the selection probabilities.

    geometric (NEXT-2, reading Q18): gamma(t) comes from the skip stream, so
    a node-update needs a selection word only when its node has ell > 1, no
    T_p compare, and under VECTOR no evaluation at all on the chain-steps
    with gamma != 0: every node term is scaled by P(gamma = 0) = (1-p)^n
    (the skip draws cost ~(1 + n p) words per chain-step, / n per node)."""
    ell = np.diff(model.fn_off).astype(np.float64)
    theta = np.diff(model.par_off).astype(np.float64)
    node_of_fn = np.repeat(np.arange(model.n), np.diff(model.fn_off))
    sel_theta = np.bincount(node_of_fn, weights=model.sel_prob * theta, minlength=model.n)
    sel_big = np.bincount(node_of_fn, weights=model.sel_prob * (theta >= 6), minlength=model.n)
    thmax = np.zeros(model.n)
    np.maximum.at(thmax, node_of_fn, theta)
    slow = (ell > 4) | (thmax > 8)                       # the generic (dense) path
    steps = np.ceil(np.log2(np.maximum(ell, 1.0)))
    decide = np.where(slow, 1.0 + 3.0 * steps, ell + 1.0)
    alu = (5.0 + decide + 2.0 * sel_theta + 2.0 + sel_big + 1.0).mean()
    fma = 5.0
    if geometric:
        p0 = (1.0 - float(model.p)) ** model.n
        needs_word = (ell > 1).astype(np.float64)
        alu = float(p0 * (5.0 * needs_word + (decide - 1.0) + 2.0 * sel_theta + 2.0 + sel_big + 1.0).mean())
        fma = float(p0 * 5.0 * needs_word.mean())
        sel_theta = p0 * (sel_theta + 1.0) - 1.0      # smem demand below: p0 (theta_sel + 1) / 32
    img_bytes = np.where(slow, 16.0 / 32 + 4.0 * steps + 16.0 + 4.0 * sel_theta + 4.0, 0.0).mean()
    return {"alu": float(alu), "fma": fma, "issue": float(alu + fma),
            "lds_wavefronts": float((sel_theta.mean() + 1.0) / 32.0), "image_bytes": float(img_bytes),
            "theta_sel": float(sel_theta.mean()), "ell": float(ell.mean()), "dense_nodes": float(slow.mean())}


def demand_bitslice(model) -> dict:
    """Algorithmic demand per node-update of the bit-sliced formulation K1b
    runs: RNG 1/4 Philox (5 LOP3 + 5 IMAD.WIDE); per node (ell-1)
    compare + ballot pairs (the selection planes) and the quad's perturbation
    flag (two min, one compare, one vote per 4 nodes); per predictor
    function, once per 32 chains, its multiplexer tree (2^c entry masks +
    2^c - 1 muxes, c = max(theta, 1)) and ~4 ops to mask it by its plane and
    commit.  (SURVEY §8(d)'s demand line -- the per-chain method -- stays the
    bench's `roofline`; this is the same work counted for the algorithm the
    kernel actually runs.)"""
    ell = np.diff(model.fn_off).astype(np.float64)
    theta = np.maximum(np.diff(model.par_off), 1).astype(np.float64)
    per_fn = (2.0 ** (theta + 1) - 1.0 + 4.0).sum() / (32.0 * model.n)
    alu = 5.0 + 2.0 * (ell - 1.0).mean() + 1.0 + per_fn
    return {"alu": float(alu), "fma": 5.0, "issue": float(alu + 5.0)}


def load_peaks() -> dict:
    """Per-SM per-clock peaks measured by microbench/peaks.cu on a B200 of this
    pool (profiles/peaks.json); the SM clock of the run scales them."""
    path = os.path.join(ROOT, "profiles", "peaks.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        t = pk["tests"]
        return {"source": "measured: profiles/peaks.json (microbench/peaks.cu, " + pk.get("when", "?") + ")",
                "alu_warp_instr_per_clk": t["LOP3 (alu)"]["warp_instr_per_clk_per_sm"],
                "fma_warp_instr_per_clk": t["IMAD (fma)"]["warp_instr_per_clk_per_sm"],
                "issue_warp_instr_per_clk": t["LOP3+IMAD (issue)"]["warp_instr_per_clk_per_sm"],
                "lds_wavefronts_per_clk": t["LDS.32 32 banks (1 wf)"]["warp_instr_per_clk_per_sm"],
                "l2_read_gbs": pk.get("l2_read_gbs")}
    # fallback: the guide's unit counts (B300_MICROARCH.md: ALU rt_SMSP = 2)
    return {"source": "guide unit counts (no profiles/peaks.json)", "alu_warp_instr_per_clk": 2.0,
            "fma_warp_instr_per_clk": 2.0, "issue_warp_instr_per_clk": 4.0, "lds_wavefronts_per_clk": 1.0,
            "l2_read_gbs": None}


def roofline(model, node_updates: float, kernel_s: float, sm_mhz: float, geometric: bool = False) -> dict:
    """Roofline of K1 in node-updates/s = min over resources of peak/demand
    (SURVEY §8(d)); frac = achieved / roofline; `achieved`/`peak` are given
    in the binding resource's unit (T ops/s or T wavefronts/s)."""
    d = demand_per_node_update(model, geometric)
    pk = load_peaks()
    hz = sm_mhz * 1e6 * SM_COUNT_B200
    res = {
        "alu": (pk["alu_warp_instr_per_clk"] * 32 * hz, d["alu"], "Tops/s"),
        "fma": (pk["fma_warp_instr_per_clk"] * 32 * hz, d["fma"], "Tops/s"),
        "issue": (pk["issue_warp_instr_per_clk"] * 32 * hz, d["issue"], "Tinstr/s"),
        "smem": (pk["lds_wavefronts_per_clk"] * hz, d["lds_wavefronts"], "Twavefronts/s"),
    }
    if d["image_bytes"] > 0 and pk.get("l2_read_gbs"):
        # generic-path nodes read their image through L1/L2 (the dense class)
        res["l2"] = (pk["l2_read_gbs"] * 1e9, d["image_bytes"], "TB/s")
    rate = node_updates / kernel_s
    per = {k: {"peak": P / 1e12, "demand_per_node_update": D, "roofline_node_updates_per_s": P / D,
               "frac": rate * D / P, "unit": U} for k, (P, D, U) in res.items()}
    bound = min(per, key=lambda k: per[k]["roofline_node_updates_per_s"])
    b = per[bound]
    return {"bound": bound if bound != "smem" else "smem", "achieved": rate * b["demand_per_node_update"] / 1e12,
            "peak": b["peak"], "unit": b["unit"], "frac": b["frac"],
            "roofline_node_updates_per_s": b["roofline_node_updates_per_s"], "achieved_node_updates_per_s": rate,
            "sm_mhz": sm_mhz, "peaks": pk, "per_resource": per, "demand": d}


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference) -- the only
# places bench.py executes oracle/.
# --------------------------------------------------------------------------
def oracle_sample(model, pred, seed: int, chains: int, steps: int, threads: int) -> tuple[float, dict]:
    from oracle import sim as osim
    from oracle import stats as ostats
    t0 = time.perf_counter()
    _, I = osim.simulate(model, pred, seed=seed, chain_ids=np.arange(chains), step0=0, burn_in=0,
                         steps=steps, threads=threads)
    _ = [ostats.window_stats(I[c], 500) for c in range(chains)]
    dt = time.perf_counter() - t0
    nu = chains * steps * model.n
    return nu / dt, {"chains": chains, "steps_per_chain": steps, "seconds": dt, "node_updates": nu}


def run_reference(args, cfg, model, pred, rank: int):
    if rank != 0:
        return
    cores = ncores()
    chains = cores
    steps = max(200, int(args.ref_steps))
    vals = []
    for i in range(args.warmup + args.steps):
        v, info = oracle_sample(model, pred, cfg.sim_seed, chains, steps, cores)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    sample = (f"{chains} chains x {steps} transitions of {cfg.key} (n={model.n}) per step, "
              f"oracle C simulator + window statistics, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": chains * steps * model.n / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(args, cfg, model),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, cfg, model) -> dict:
    return {
        "workload": f"{cfg.key}: n={model.n} PBN, ell~U{{{cfg.ell[0]}..{cfg.ell[1]}}}, "
                    f"theta~U{{{cfg.theta[0]}..{cfg.theta[1]}}}, p={cfg.p}, "
                    f"{args.chains} chains x ({args.burn_in} burn-in + {args.window} recorded) "
                    f"transitions, fused c1/n01/n10/first-last, batch kappa={cfg.batch}, bits, totals",
        "chains_per_gpu": args.chains, "burn_in": args.burn_in, "window": args.window,
        "batch": cfg.batch, "n": model.n, "functions": int(model.nf),
        "density": float(model.par_off[-1]) / model.n, "seed": cfg.sim_seed,
        "semantics": "VECTOR, geometric-skip stream (NEXT-2)" if getattr(args, "geometric", False) else "VECTOR",
        "l2": "256 MiB buffer written between timed steps",
    }


# --------------------------------------------------------------------------
def run_sweep(args, cfg, model, pred):
    """BASELINE config C5: node-updates/s and ALU-roofline fraction versus chain
    count (one JSON line per chain count; not the driver's bench line)."""
    import torch
    import paper_1508_07828_b200 as pbn
    torch.cuda.set_device(0)
    pm = pbn.pbn_load(model)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    sweep = cfg.extra.get("chain_sweep", (1, 64, 1024, 16384))
    for chains in sweep:
        out = pbn.alloc_outputs(pm, chains, args.window, batch=cfg.batch, emit_bits=True)

        def one():
            pbn.pbn_simulate(pm, out, n_chains=chains, steps=args.window, burn_in=args.burn_in,
                             batch=cfg.batch, seed=cfg.sim_seed, pred=pred, init=True, emit_bits=True,
                             layout=args.layout, stream=stream)
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            one()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        t = statistics.median(ms) / 1e3
        nu = chains * (args.burn_in + args.window) * model.n
        rf = roofline(model, nu, t, 1965.0)
        print(json.dumps({"sweep": cfg.key, "chains": chains, "n": model.n, "kernel": pbn.pbn_last_kernel(),
                          "steps_per_chain": args.burn_in + args.window,
                          "node_updates_per_s": nu / t, "chain_steps_per_s": chains * (args.burn_in + args.window) / t,
                          "ms": t * 1e3, "ms_best": min(ms) * 1.0, "roofline_frac": rf["frac"], "bound": rf["bound"],
                          "roofline_node_updates_per_s": rf["roofline_node_updates_per_s"],
                          "image_bytes": int(pm.info.image_bytes)}), flush=True)
        del out
    pm.close()


# --------------------------------------------------------------------------
def run_protocol(args):
    """The whole method on the GPU through pbn_run (Algorithm 3, then 4 or 5,
    the paper's unit of work, Table 1): C2 with the two-state rule
    (BASELINE config 2), C3 with Skart (config 3).  Reports the decisions, the
    pooled sample, the transitions simulated and the device time; not the
    driver's bench line."""
    import torch
    import paper_1508_07828_b200 as pbn
    torch.cuda.set_device(0)
    for key in args.protocol.split(","):
        cfg = CONFIGS[key]
        model, pred = config_model(key), config_predicate(key)
        pm = pbn.pbn_load(model)
        x = cfg.extra
        if key == "C3":
            kw = dict(method=1, omega=cfg.chains, psi0=cfg.burn_in, rhat_threshold=1.1, h_star=x["h_star"],
                      alpha_conf=x["alpha_conf"], seed=cfg.sim_seed, pred=pred, max_steps=1 << 22)
        else:
            kw = dict(method=0, omega=cfg.chains, psi0=x.get("psi0", 1000), rhat_threshold=x.get("rhat_threshold", 1.1),
                      r=x.get("r", 0.01), s=x.get("s", 0.95), eps=x.get("eps", 1e-10), seed=cfg.sim_seed, pred=pred,
                      max_steps=1 << 24)
        pbn.pbn_run(pm, **kw)  # warm-up
        torch.cuda.synchronize()
        dts = []
        for _ in range(3):  # wall clock with host statistics inside: the median of three runs
            t0 = time.perf_counter()
            st, res, err = pbn.pbn_run(pm, **kw)
            torch.cuda.synchronize()
            dts.append(time.perf_counter() - t0)
        dt = sorted(dts)[1]
        nu = cfg.chains * res.steps_per_chain * model.n
        cpu = None
        if key == "C2" and not args.no_cpu_baseline:
            # cpu_baseline leg: the oracle's Algorithm 3 + 4 on the same inputs
            from oracle import driver as odr
            t1 = time.perf_counter()
            o = odr.parallel_two_state(model, pred, cfg.sim_seed, cfg.chains, kw["psi0"], kw["rhat_threshold"],
                                       kw["r"], kw["s"], kw["eps"], kw["max_steps"], threads=ncores())
            cpu = {"seconds": time.perf_counter() - t1, "cores": ncores(), "kind": "oracle",
                   "same_decisions": (o.psi, o.sample_size, o.M, o.N) == (res.psi, res.sample_size, res.M, res.N)}
        print(json.dumps({"protocol": key, "cpu_baseline": cpu, "method": "skart" if kw["method"] == 1 else "two-state", "status": st,
                          "err": err, "omega": cfg.chains, "psi": res.psi, "gr_iterations": res.gr_iterations,
                          "rhat": res.rhat, "extensions": res.extensions, "M": res.M, "N": res.N,
                          "sample_size": res.sample_size, "steps_per_chain": res.steps_per_chain,
                          "estimate": res.estimate, "ci": [res.ci_lo, res.ci_hi], "seconds": dt,
                          "seconds_runs": dts,
                          "node_updates_per_s": nu / dt,
                          "note": "wall time of pbn_run (GPU kernels + host statistics + D2H decision reads)"}),
              flush=True)
        pm.close()


# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--chains", type=int, default=None)
    ap.add_argument("--burn-in", type=int, default=None)
    ap.add_argument("--window", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-steps", type=int, default=2500)
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--schedule", type=int, default=0, help="0 auto, 1 CTA per group, 2 persistent")
    ap.add_argument("--chunk", type=int, default=0, help="persistent chunk steps (0 auto)")
    ap.add_argument("--cluster", type=int, default=0, help="cluster_size (0 auto)")
    ap.add_argument("--layout", type=int, default=0,
                    help="PBN_LAYOUT_*: 0 auto, 1 chain lanes (K1/K1c), 2 node lanes (K1n), 3 bit-sliced (K1b)")
    ap.add_argument("--sweep", action="store_true", help="C5 chain-count sweep (one line per count)")
    ap.add_argument("--e2e-steps", type=int, default=3, help="timed end-to-end (host buffer) iterations")
    ap.add_argument("--protocol", default="",
                    help="time the whole method (pbn_run) on C2 and/or C3, e.g. --protocol C2,C3")
    ap.add_argument("--geometric", action="store_true",
                    help="geometric-skip perturbation stream (NEXT-2, PBN_PERTURB_GEOMETRIC)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)

    if args.sweep and args.config == "C4":
        args.config = "C5"
    cfg = CONFIGS[args.config]
    args.chains = args.chains or cfg.chains
    args.burn_in = cfg.burn_in if args.burn_in is None else args.burn_in
    args.window = cfg.steps if args.window is None else args.window
    model, pred = config_model(args.config), config_predicate(args.config)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.sweep:
        run_sweep(args, cfg, model, pred)
        return
    if args.protocol:
        run_protocol(args)
        return
    if args.impl == "reference":
        run_reference(args, cfg, model, pred, rank)
        return

    import torch
    import paper_1508_07828_b200 as pbn

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    pm = pbn.pbn_load(model, geometric=args.geometric)
    chains, burn_in, window, batch = args.chains, args.burn_in, args.window, cfg.batch
    chain_base = rank * chains                    # disjoint global chain ids per rank
    out = pbn.alloc_outputs(pm, chains, window, batch=batch, emit_bits=True)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def one_step():
        pbn.pbn_simulate(pm, out, n_chains=chains, chain_base=chain_base, steps=window,
                         burn_in=burn_in, batch=batch, seed=cfg.sim_seed, pred=pred, init=True,
                         emit_bits=True, groups_per_cta=args.groups, warps_per_group=args.warps,
                         schedule=args.schedule, chunk_steps=args.chunk, layout=args.layout,
                         cluster_size=args.cluster, stream=stream)

    for _ in range(args.warmup):
        one_step()
        flush.fill_(1)
    torch.cuda.synchronize()
    kernel_name = {"K1b": "bitslice_kernel (K1b)", "K1b-global": "bitslice_kernel (K1b, global image)",
                   "K1bc": "bitslice_kernel (K1bc, cluster)",
                   "K1": "traj_kernel (K1)", "K1-global": "traj_kernel (K1, global image)",
                   "K1c": "traj_cluster_kernel (K1c)", "K1n": "traj_nodepar_kernel (K1n)"}.get(
        pbn.pbn_last_kernel(), pbn.pbn_last_kernel())

    clocks = ClockSampler(local_rank)
    if rank == 0:
        clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        ev[k][0].record(stream)
        one_step()
        ev[k][1].record(stream)
        flush.fill_(k)
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    if dist:  # device-timed region: max over ranks (paper_1508_07828_b200.parallel)
        total_ms = pbn.parallel.max_over_ranks(total_ms)
    clk = clocks.stop() if rank == 0 else None

    node_updates_per_step = chains * (burn_in + window) * model.n
    value = world * node_updates_per_step * args.steps / (total_ms / 1e3)
    chain_steps = world * chains * (burn_in + window) * args.steps / (total_ms / 1e3)

    # ---- roofline of the dominant kernel (K1 traj_kernel; one launch per step) ----
    avg_kernel_s = statistics.mean(kern_ms) / 1e3
    sm_mhz = None
    if clk and clk.get("sm_mhz"):
        sm_mhz = float(clk["sm_mhz"])           # SM clock sampled during the timed region
    if not sm_mhz:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                sm_mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
        except Exception:
            sm_mhz = 1965.0
    rf = roofline(model, node_updates_per_step, avg_kernel_s, sm_mhz, args.geometric)
    if pbn.pbn_last_kernel() in ("K1b", "K1b-global", "K1bc"):
        db = demand_bitslice(model)
        alu_peak = rf["per_resource"]["alu"]["peak"] * 1e12
        rate = node_updates_per_step / avg_kernel_s
        rf["kernel_algorithm"] = {
            "kernel": "K1b", "demand_per_node_update": db,
            "alu_roofline_node_updates_per_s": alu_peak / db["alu"], "alu_frac": rate * db["alu"] / alu_peak,
            "note": "the bit-sliced algorithm needs fewer ALU ops per node-update than SURVEY 8(d)'s per-chain "
                    "demand line; roofline.frac keeps 8(d)'s line, this is K1b's own"}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_C4.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            if tj.get("chains") == chains and tj.get("steps") == burn_in + window:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e: same workload through the public API with HOST buffers ----
    e2e = None
    if rank == 0 or True:
        rng = np.random.default_rng(cfg.sim_seed)
        host_state = torch.from_numpy(
            rng.integers(0, 2**32, size=(chains, pm.state_words), dtype=np.uint64)
            .astype(np.uint32).view(np.int32)).pin_memory()
        res_host = {k: torch.empty(tuple(getattr(out, k).shape), dtype=getattr(out, k).dtype).pin_memory()
                    for k in ["state", "c1", "n01", "n10", "first_last", "batch_sums", "bits", "totals"]}
        h2d = host_state.numel() * 4
        d2h = sum(t.numel() * t.element_size() for t in res_host.values())

        def e2e_step():
            out.state.copy_(host_state, non_blocking=True)
            pbn.pbn_simulate(pm, out, n_chains=chains, chain_base=chain_base, steps=window,
                             burn_in=burn_in, batch=batch, seed=cfg.sim_seed, pred=pred, init=False,
                             emit_bits=True, warps_per_group=args.warps, layout=args.layout,
                             cluster_size=args.cluster, stream=stream)
            for k, t in res_host.items():
                t.copy_(getattr(out, k), non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e2e_ms = []
        for _ in range(max(1, args.e2e_steps)):
            flush.fill_(7)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1)
            if dist:
                ems = pbn.parallel.max_over_ranks(ems)
            e2e_ms.append(ems)
        ems = statistics.median(e2e_ms)
        e2e = {"value": world * node_updates_per_step / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": len(e2e_ms),
               "ms_per_step_median": ems, "ms_per_step_best": min(e2e_ms),
               "path": "pinned host state -> pbn_simulate -> all outputs to pinned host (median of steps)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = ncores()
        steps_s = 250_000 if model.n >= 1000 else 1_000_000  # ~10-20 s of oracle work
        v, info = oracle_sample(model, pred, cfg.sim_seed, cores, steps_s, cores)
        # the same oracle on one core (one chain), a fifth of the per-chain steps
        v1, info1 = oracle_sample(model, pred, cfg.sim_seed, 1, max(1, steps_s // 5), 1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{info['chains']} chains x {info['steps_per_chain']} transitions of "
                         f"{cfg.key} ({info['seconds']:.1f} s wall, one thread per chain)",
               "single_core": {"value": v1, "unit": UNIT, "cores": 1,
                               "sample": f"1 chain x {info1['steps_per_chain']} transitions "
                                         f"({info1['seconds']:.1f} s)"},
               "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "chain_steps_per_s": chain_steps,
            "config": workload_config(args, cfg, model),
            "roofline": {"bound": rf["bound"], "achieved": rf["achieved"], "peak": rf["peak"], "unit": rf["unit"],
                         "frac": rf["frac"], "traffic": traffic,
                         "roofline_node_updates_per_s": rf["roofline_node_updates_per_s"],
                         "peak_basis": f"{rf['peaks']['source']}; x 32 lanes x {SM_COUNT_B200} SMs x "
                                       f"{sm_mhz:.0f} MHz (SM clock sampled in the timed region); "
                                       "roofline = min over resources of peak / demand (SURVEY 8(d))",
                         "per_resource": rf["per_resource"], "demand": rf["demand"],
                         "kernel_algorithm": rf.get("kernel_algorithm"),
                         "kernel": kernel_name, "kernel_ms_mean": statistics.mean(kern_ms),
                         "kernel_ms_median": statistics.median(kern_ms), "kernel_ms_best": min(kern_ms)},
            "value_best": node_updates_per_step * world / (min(kern_ms) / 1e3),
            "value_median": node_updates_per_step * world / (statistics.median(kern_ms) / 1e3),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
