#!/usr/bin/env python
"""bench.py -- MP GEMM throughput on B200 (BASELINE.json metric: MP mul-adds/s,
n^3/t, and % of the INT32 IMAD roofline on the leaf GEMM).

Workload (N = 1): BASELINE config 2 -- square MP GEMM n = 1024 at 256 bits, entries
uniform in [-1, 1) with all mantissa bits random (seeded), Winograd with recursion
cutoff n_min = 64 (depth 4, 2401 leaves of 64^3).  One step = one fast_mul of the
resident operands.  --algo block|strassen|winograd|simple selects the other arms.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (one process per GPU; started without torchrun, bench.py re-launches itself as N
ranks): the 7^d leaf products are sharded across ranks (each rank does the pre-additions
for its own leaves from replicated A and B); the leaf kernel's epilogue stores every
product row straight into the buffer of the rank that owns it (peer memory over NVLink,
CUDA IPC) and each rank post-adds its own rows of C.  Timing: CUDA events around each step
on the launching stream, an L2 flush (256 MiB write) between steps, barrier +
synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
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

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
IMAD_PER_CLK_PER_SM = 64  # INT32 IMAD issue rate of the FMA pipe (Nsight profiling guide; tools/microbench_pipes.cu)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--algo", default="winograd", choices=["simple", "block", "strassen", "winograd"])
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--n-min", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-precision-sweep", action="store_true",
                    help="skip the leaf-roofline sweep at 512 / 1024 bits (same n, algorithm, n_min)")
    ap.add_argument("--no-lu", action="store_true", help="skip the config-5 LU leg")
    ap.add_argument("--probe-world", action="store_true",
                    help="print this rank's (rank, world) as JSON and exit before touching CUDA (launcher test)")
    ap.add_argument("--cfg4", action="store_true", help="(default) time config 4 (n=4096 @1024)")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-4 leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the config-1 / config-3 legs")
    ap.add_argument("--shard", choices=["auto", "a2a", "gather", "replicas"], default="auto",
                    help="N>1: auto = leaf shards whose leaf epilogue stores the product rows into their owners' "
                         "buffers over peer memory (CUDA IPC, NVLink), then a row-owned combine (Strassen/Winograd), "
                         "or row shards (Simple/Block) (strong scaling); a2a = the same with an NCCL all-to-all; "
                         "gather = leaf shards + all-gather + replicated combine; replicas = independent copies (weak)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def issued_imad_eq_per_madd(L, bits):
    """IMAD-equivalents the leaf issues per multiply-add: the short product (mp_arith.cuh mul_high_g)
    when the precision fills its limbs, the full product otherwise."""
    products = (L * L + 3 * L - 2) // 2 if (bits == 32 * L and L >= 3) else L * L
    return 2 * products


def measured_peaks():
    try:
        return json.loads(PEAKS_FILE.read_text())
    except Exception:
        return {}


def nbytes_soa(n_elems: int, limbs: int) -> int:
    return n_elems * (4 * limbs + 4 + 1)


# ---------------------------------------------------------------------------
def host_info():
    """lscpu model name and nproc of the host the CPU arm ran on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_inputs(args, s):
    """The workload's inputs made by the ORACLE's generator (oracle/mp_oracle.c, the same
    Prng64 stream as the product's gen_uniform_full: tests/test_cpu_host.py), cut to the
    top-left s x s blocks -- the reference arm never maps libmpgpu.so."""
    from oracle import oracle as O
    out = []
    for seed in (1, 2):
        full = O.gen_full(0, args.n, args.n, seed, args.bits)
        idx = (np.arange(s)[:, None] * args.n + np.arange(s)[None, :]).reshape(-1)
        out.append(O.OMat(s, s, args.bits, full.limbs[:, idx], full.exp[idx], full.sign[idx]))
    return out


def run_reference(args, rank: int):
    """The reference's own CPU implementation (oracle/_ref: the unmodified mpmm
    headers compiled against system MPFR), all host threads, bounded sample.
    Imports only oracle/ (never the product package)."""
    if rank != 0:
        return
    from oracle import oracle as O
    s, nmin_s = sample_shape(args)
    oa, ob = oracle_inputs(args, s)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        O.gemm_replicas(args.algo, nmin_s, oa, ob, threads)
    times = []
    for _ in range(args.steps):
        _, sec = O.gemm_replicas(args.algo, nmin_s, oa, ob, threads)
        times.append(sec)
    total = sum(times)
    value = threads * s ** 3 * len(times) / total
    sample = sample_desc(args, s, nmin_s, threads)
    line = {
        "metric": "MP mul-adds/s (n^3/t, classical-equivalent)", "value": value, "unit": "madd/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": f"mp{args.bits} (MPFR)",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(args),
        "sample": {"shape": [s, s, s], "n_min": nmin_s if args.algo != "simple" else None, "algorithm": args.algo,
                   "replicas": threads, "what": sample},
        "host": host_info(),
        "cpu_baseline": {"value": value, "unit": "madd/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "madd/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def sample_shape(args):
    """Bounded CPU sample of the workload: the same algorithm at n/4 with the
    cutoff scaled by 1/4, i.e. the same recursion depth and op-count ratio."""
    if args.algo in ("strassen", "winograd"):
        s = max(args.n // 4, 1)
        return s, max(args.n_min // 4, 1)
    return max(args.n // 4, 1), args.n_min


def sample_desc(args, s, nmin_s, threads):
    what = f"{args.algo}(n_min={nmin_s})" if args.algo != "simple" else "simple"
    return (f"SAMPLE, not the full workload: {threads} thread(s) each running the reference's {what} on the "
            f"{s}x{s} top-left blocks of the workload inputs ({args.bits}-bit; same recursion depth and op-count "
            f"ratio as n={args.n}, n_min={args.n_min}); value = threads * {s}^3 / wall time of the multiplies. "
            f"The full-size single-core reference timing of this workload is in profiles/ (r02_ref_fullsize_*.json)")


def workload_config(args, world=None):
    world = args.gpus if world is None else world
    return {"workload": f"BASELINE config 2: MP GEMM n={args.n} @{args.bits}-bit, {args.algo}"
                        + (f" n_min={args.n_min}" if args.algo != "simple" else ""),
            "n": args.n, "bits": args.bits, "algorithm": args.algo, "n_min": args.n_min,
            "inputs": "uniform [-1,1) full-mantissa, seeds 1/2 (Prng64)",
            "l2": "flushed between timed steps (256 MiB write) and working set > L2",
            "parallelism": (f"{args.shard} x{world}" if world > 1 else "single GPU")}


# ---------------------------------------------------------------------------
def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` started without torchrun: re-launch this command as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.probe_world:
        # one write(2) per line: the ranks share stdout and print() may split the line and its newline
        os.write(1, (json.dumps({"rank": rank, "world": world, "local_rank": local, "gpus": args.gpus}) + "\n").encode())
        return
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)
    import torch
    import paper_1410_1599_b200 as P
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P.set_device(local)
    stream = torch.cuda.current_stream()
    P.set_stream(stream.cuda_stream)

    ctx = P.PrecisionContext(args.bits)
    algo = P.Algorithm[args.algo]
    param = args.n_min if algo != P.Algorithm.simple else 0
    n = args.n
    a = P.gen_uniform_full(n, n, 1, ctx)
    b = P.gen_uniform_full(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    dc = P.DeviceMatrix(n, n, ctx)
    L = P.nlimbs_for(args.bits)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    from paper_1410_1599_b200 import shard
    runner = shard.make_runner(algo, param, da, db, dc, rank, world, mode=args.shard) if world > 1 else None

    def step():
        if runner is not None:
            return runner()
        return P.gemm_into(algo, param, da, db, dc)

    total_ms, leaf_ms, launches, st, clocks = timed_steps(args, torch, dist, stream, flush, step, local)
    # every rank works on one n^3 problem together (N > 1: leaf shards); weak scaling
    # is reported via replicas of the problem per rank -- see shard.make_runner
    problems = world if (runner is not None and runner.replicated) else 1
    value = problems * n ** 3 * args.steps / (total_ms * 1e-3)

    # correctness guard on the timed output (outside the timed region)
    guard = check_output(args, P, torch, dist, algo, param, a, b, da, db, dc, runner, rank, world)

    e2e_res = None
    if world > 1 and not args.no_e2e:
        e2e_res = e2e_dist(args, P, torch, dist, a, b, da, db, dc, runner, rank, world)
    big = None
    if not args.no_cfg4:
        big = cfg4_leg(args, P, torch, dist, stream, flush, local, rank, world)
    others = None
    if world == 1 and not args.no_configs:
        others = other_configs(args, P, torch, stream, flush, local)

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (leaf GEMM): algorithmic IMAD-equivalents
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    leaf_avg_ms = float(np.mean(leaf_ms))
    imad_eq = st.leaf_madds * 2 * L * L
    achieved = imad_eq / (leaf_avg_ms * 1e-3) / 1e12
    peak = IMAD_PER_CLK_PER_SM * sms * sm_max * 1e6 / 1e12
    prof = ROOT / "profiles" / "r01_leaf_traffic.json"
    traffic = None
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{args.algo}_{n}_{args.bits}")
        except Exception:
            traffic = None
    roof = {"bound": "imad", "achieved": achieved, "peak": peak, "unit": "TIOP/s (IMAD-eq)",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": "mpg::gemm_leaf_kernel", "leaf_ms": leaf_avg_ms, "leaf_madds_per_launch": st.leaf_madds,
            "imad_eq_per_madd": 2 * L * L,
            "peak_basis": f"{IMAD_PER_CLK_PER_SM} IMAD/clk/SM x {sms} SMs x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"}
    if clocks.get("sm_mhz"):
        roof["frac_at_measured_clock"] = achieved / (IMAD_PER_CLK_PER_SM * sms * clocks["sm_mhz"] * 1e6 / 1e12)
    # the kernel issues the SHORT product when p == 32 L ((L^2 + 3L - 2)/2 limb products, one
    # IMAD.WIDE.U32 = 2 IMAD-eq each): the share of the IMAD pipe those issued products hold
    issued = issued_imad_eq_per_madd(L, args.bits)
    roof["issued_imad_eq_per_madd"] = issued
    roof["frac_issued"] = roof["frac"] * issued / (2 * L * L)

    line = {
        "metric": "MP mul-adds/s (n^3/t, classical-equivalent)", "value": value, "unit": "madd/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if problems > 1 else "strong", "vs_baseline": None,
        "dtype": f"mp{args.bits} (u32 limbs, IMAD)", "data": "synthetic", "config": workload_config(args, world),
        "ops_per_step": {"mul": st.mul, "addsub": st.addsub, "leaf_madds": st.leaf_madds, "depth": st.depth},
        "phase_ms": {"preadd": st.preadd_ms, "leaf": st.leaf_ms, "postadd": st.postadd_ms},
        "roofline": roof, "clocks": clocks, "gpu_launches": launches, "check": guard,
    }
    if runner is not None:
        line["config"]["runner"] = runner.mode

    if not args.no_e2e and world == 1:
        line["e2e"] = e2e(args, P, torch, a, b, algo, param, ctx, L)
    elif not args.no_e2e:
        line["e2e"] = e2e_res
    if big is not None:
        line["cfg4"] = big
    if others is not None:
        line["configs_1_3"] = others
    if not args.no_precision_sweep and world == 1:
        line["leaf_roofline_by_bits"] = precision_sweep(args, P, torch, IMAD_PER_CLK_PER_SM * sms * sm_max * 1e6 / 1e12)
    if not args.no_lu and world == 1:
        line["lu"] = lu_leg(args, P, torch, stream, flush, peak)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args, P, a, b)
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def timed_steps(args, torch, dist, stream, flush, step, local, steps=None, warmup=None):
    """W untimed warm-up steps, then K steps each bracketed by CUDA events on the launching
    stream, an L2 flush between steps, barrier + synchronize on both sides; max over ranks."""
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times, leaf_ms, launches, st = [], [], 0, None
    with ClockSampler(local) as clk:
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            st = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            leaf_ms.append(st.leaf_ms)
            launches += st.launches
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = float(sum(times))
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    return total_ms, leaf_ms, launches, st, clk.summary()


def normwise_log2(P, x, ref, a, b):
    """log2( max|x - ref| / (max|A| max|B|) ), differences formed in MP on the device."""
    d = np.abs(P.sub(x, ref).to_float())
    num = float(d.max())
    den = float(np.abs(a.to_float()).max()) * float(np.abs(b.to_float()).max())
    return float(np.log2(num / den)) if num > 0 else float("-inf")


def check_output(args, P, torch, dist, algo, param, a, b, da, db, dc, runner, rank, world):
    """Guard on the benchmarked product (not timed).  N = 1: sampled rows of C against the
    Block product of the same rows (bit-exact for Simple / Block; for Strassen / Winograd
    within the north-star normwise bound 4 n^log2(7) 2^-p).  N > 1: every rank recomputes
    the product on its own GPU with the single-GPU path and compares the rows of C it owns
    bit for bit; mismatches are summed over ranks."""
    import math
    n = a.rows()
    if runner is None:
        rows = sorted({0, n // 3, n // 2, n - 1})
        ctx = a.ctx()
        got = dc.download()
        idx = (np.asarray(rows)[:, None] * n + np.arange(n)[None, :]).reshape(-1)
        gr = P.Matrix(len(rows), n, ctx, got.limbs[:, idx], got.exp[idx], got.sign[idx])
        ar = P.Matrix(len(rows), n, ctx, a.limbs[:, idx], a.exp[idx], a.sign[idx])
        blk = P.block_mul(ar, b, max(1, args.n_min), ctx)
        if algo in (P.Algorithm.simple, P.Algorithm.block):
            same = P.identical(gr, blk if algo == P.Algorithm.block else P.simple_mul(ar, b, ctx))
            return {"rows": rows, "vs": "same algorithm on the sampled rows", "bit_exact": bool(same), "ok": bool(same)}
        err = normwise_log2(P, gr, blk, a, b)
        bound = math.log2(4.0) + math.log2(7) * math.log2(n) - args.bits
        return {"rows": rows, "vs": "Block rows, normwise", "log2_err": err, "log2_bound": bound,
                "ok": bool(err <= bound)}
    ref = P.DeviceMatrix(n, n, a.ctx())
    P.gemm_into(algo, param, da, db, ref)
    own = getattr(runner, "c_rows", None)
    if own is None or getattr(runner, "replicated", False) or runner.__class__.__name__ == "_FastSharded":
        own = list(range(n))
    elif runner.__class__.__name__ == "_RowSharded":
        own = list(range(runner.shard.lo, min(runner.shard.hi, n)))
    got, want = dc.download(), ref.download()
    ref.free()
    idx = (np.asarray(own, dtype=np.int64)[:, None] * n + np.arange(n)[None, :]).reshape(-1) if own else \
        np.zeros(0, np.int64)
    bad = int(np.count_nonzero((got.exp[idx] != want.exp[idx]) | (got.sign[idx] != want.sign[idx]) |
                               np.any(got.limbs[:, idx] != want.limbs[:, idx], axis=0)))
    t = torch.tensor([bad, len(own)], device="cuda", dtype=torch.int64)
    dist.all_reduce(t)
    return {"vs": "single-GPU product of the same inputs on every rank, owned rows, bit for bit",
            "mismatched_elements": int(t[0].item()), "rows_checked": int(t[1].item()), "ok": int(t[0].item()) == 0}


def cfg4_leg(args, P, torch, dist, stream, flush, local, rank, world):
    """north star's scaling workload (BASELINE config 4): n = 4096 at 1024 bits, Winograd
    n_min 512 (depth 3, 343 leaves of 512^3) sharded the same way; 1 warm-up + 1 timed step."""
    from paper_1410_1599_b200 import shard
    ctx = P.PrecisionContext(1024)
    n, nmin = 4096, 512
    a = P.gen_uniform_full(n, n, 1, ctx)
    b = P.gen_uniform_full(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    dc = P.DeviceMatrix(n, n, ctx)
    algo = P.Algorithm.winograd
    runner = shard.make_runner(algo, nmin, da, db, dc, rank, world, mode=args.shard) if world > 1 else None

    def step():
        return runner() if runner is not None else P.gemm_into(algo, nmin, da, db, dc)

    total_ms, leaf_ms, launches, st, clocks = timed_steps(args, torch, dist, stream, flush, step, local, 1, 1)
    L = P.nlimbs_for(1024)
    out = {"workload": "BASELINE config 4: MP GEMM n=4096 @1024-bit, winograd n_min=512 (depth 3)",
           "value": n ** 3 / (total_ms * 1e-3), "unit": "madd/s", "ms_per_step": total_ms, "steps": 1, "warmup": 1,
           "leaf_ms_rank0": float(np.mean(leaf_ms)), "leaf_madds_rank0": st.leaf_madds,
           "imad_eq_per_madd": 2 * L * L, "runner": getattr(runner, "mode", "single GPU"), "clocks": clocks}
    if world == 1:
        # the same product at the cutoff chosen from the measured leaf throughput (deeper recursion,
        # top levels depth-first beyond the scratch budget) -- an extension, reported beside
        nm, depth, model_ms = P.choose_n_min(algo, 1024, n, n, n)
        P.gemm_into(algo, P.AUTO_NMIN, da, db, dc)
        sa = P.gemm_into(algo, P.AUTO_NMIN, da, db, dc)
        out["auto_n_min"] = {"n_min": nm, "depth": depth, "model_ms": model_ms, "device_ms": sa.device_ms,
                             "leaf_ms": sa.leaf_ms, "value": n ** 3 / (sa.device_ms * 1e-3)}
        ref = ROOT / "profiles" / "r02_ref_cfg4_extrapolated.json"
        if ref.exists():
            try:
                out["cpu_reference_extrapolated"] = json.loads(ref.read_text())
            except Exception:
                pass
    if hasattr(runner, "close"):
        if dist:
            dist.barrier()
        runner.close()
    for x in (da, db, dc):
        x.free()
    return out


def other_configs(args, P, torch, stream, flush, local):
    """BASELINE configs 1 and 3 on the same GPU (CUDA events, min of 5 after 2 warm-ups): cfg1 128^3
    @128 bits -- Simple, Block 32, Strassen / Winograd cutoff 32 -- and cfg3 1001 x 777 x 1537 @512
    bits, config-3 inputs, Winograd with pad-only odd handling at cutoffs 32 and 64.  Bit-exact
    parity of these shapes is pinned by the test suite (tests/test_gpu_fullsize_hash.py holds the
    compiled reference's SHA-256 of both cfg3 products); here each product is also checked against
    the GPU Block product of the same operands (normwise bound for the fast algorithms)."""
    import math
    out = {}
    cases = [("cfg1", 128, 128, 128, 128, P.gen_uniform_full, [("simple", 0), ("block", 32), ("strassen", 32),
                                                               ("winograd", 32)]),
             ("cfg3", 1001, 777, 1537, 512, P.gen_scaled, [("winograd", 32), ("winograd", 64)])]
    for name, m, l, n, bits, gen, algos in cases:
        ctx = P.PrecisionContext(bits)
        a, b = gen(m, l, 1, ctx), gen(l, n, 2, ctx)
        da, db = a.to_device(), b.to_device()
        dc, ref = P.DeviceMatrix(m, n, ctx), P.DeviceMatrix(m, n, ctx)
        P.gemm_into(P.Algorithm.block, 32, da, db, ref)
        refh = ref.download()
        res = []
        for alg, param in algos:
            algo = P.Algorithm[alg]
            for _ in range(2):
                P.gemm_into(algo, param, da, db, dc)
            best = min((P.gemm_into(algo, param, da, db, dc) for _ in range(5)), key=lambda x: x.device_ms)
            got = dc.download()
            if alg == "block":
                ok, err = P.identical(got, refh), None
            else:
                err = normwise_log2(P, got, refh, a, b)
                ok = err <= math.log2(4.0) + math.log2(7) * math.log2(max(m, l, n)) - bits
            res.append({"algorithm": alg, "n_min": param, "device_ms": best.device_ms, "leaf_ms": best.leaf_ms,
                        "madd_per_s": m * l * n / (best.device_ms * 1e-3), "depth": best.depth,
                        "check": "bit-identical to Block" if alg == "block" else
                        {"log2_normwise_vs_block": err, "ok": bool(ok)}})
        out[name] = {"shape": [m, l, n], "bits": bits, "runs": res}
        for x in (da, db, dc, ref):
            x.free()
    return out


def lu_leg(args, P, torch, stream, flush, leaf_peak_tiops):
    """BASELINE config 5(a): MP LU with partial pivoting, n = 2048 at 256 bits, Winograd Schur
    update K = 64 (alpha 2, n_min 32), uniform [-1,1) full-mantissa A, b = A*1.  Device time
    (CUDA events inside mpgpu_lu_blocked), the Schur leaf roofline, e2e through the C-ABI with
    host buffers (upload, factorisation, download), the solve's forward error formed in MP on
    the device, and the compiled reference's pivot-free lu_blocked on one core at n = 256,
    extrapolated by n^3."""
    import ctypes as C
    from paper_1410_1599_b200 import _lib as PL
    try:
        n, bits, K, nmin = 2048, 256, 64, 32
        ctx = P.PrecisionContext(bits)
        L = P.nlimbs_for(bits)
        A = P.gen_uniform_full(n, n, 11, ctx)
        cfg = P.BlockLUConfig(K, P.Algorithm.winograd, nmin)
        work = P.DeviceMatrix(n, n, ctx)
        src = A.to_device()
        piv = np.zeros(n, np.int64)
        zp = C.c_int64(0)
        dev_ms, leaf_ms, leaf_madds, launches = [], [], 0, 0
        for rep in range(4):
            PL.lib.mpgpu_copy_device(work._h, C.c_void_p(work.data_ptr), C.c_void_p(src.data_ptr),
                                     C.c_size_t(work.nbytes))
            flush.zero_()
            torch.cuda.synchronize()
            s = PL.MpgpuStats()
            rc = PL.lib.mpgpu_lu_blocked(work._h, C.byref(work.m), K, int(P.Algorithm.winograd), nmin, 1,
                                         piv.ctypes.data_as(C.c_void_p), C.byref(zp), C.byref(s))
            if rc:
                raise RuntimeError(f"mpgpu_lu_blocked rc={rc}")
            if rep:
                dev_ms.append(s.device_ms)
                leaf_ms.append(s.leaf_ms)
                leaf_madds = s.leaf_madds
                launches = s.launches
        # e2e: the drop-in's call sequence (include/mpmm_gpu.hpp lu_blocked) with pinned host
        # SoA buffers: mpgpu_upload, mpgpu_lu_blocked, mpgpu_download of the packed factors
        def pinned(x):
            lim = torch.empty(x.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
            ex = torch.empty(x.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
            sg = torch.empty(x.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
            lim[:], ex[:], sg[:] = x.limbs, x.exp, x.sign
            return P.Matrix(x.rows(), x.cols(), x.ctx(), lim, ex, sg)
        ha, hf = pinned(A), pinned(A)
        e2e = []
        for rep in range(3):
            # the factorisation is in place: restore the input outside the timed region
            hf.limbs[:], hf.exp[:], hf.sign[:] = ha.limbs, ha.exp, ha.sign
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = PL.lib.mpgpu_lu_blocked_host(work._h, bits, n, hf.limbs.ctypes.data_as(C.c_void_p),
                                              hf.exp.ctypes.data_as(C.c_void_p), hf.sign.ctypes.data_as(C.c_void_p),
                                              hf.nlimbs, K, int(P.Algorithm.winograd), nmin, 1,
                                              piv.ctypes.data_as(C.c_void_p), C.byref(zp), None)
            if rc:
                raise RuntimeError(f"mpgpu_lu_blocked_host rc={rc}")
            if rep:
                e2e.append(time.perf_counter() - t0)
        e2e_ms = float(np.mean(e2e)) * 1e3
        f = P.LUFactors(n, hf, piv.copy())
        ones = P.from_ints(np.ones(n, np.int64), ctx)
        bvec = P.mat_vec_mul(A, ones, ctx)
        t0 = time.perf_counter()
        x = P.lu_solve(f, bvec, ctx, exact=False)
        solve_ms = (time.perf_counter() - t0) * 1e3
        fe = P.max_rel_error_solution(x, ones)
        fwd = float(np.abs(fe.max_rel.to_float()).max())
        schur_tiops = leaf_madds * 2 * L * L / (float(np.mean(leaf_ms)) * 1e-3) / 1e12
        out = {"workload": "BASELINE config 5(a): LU with partial pivoting n=2048 @256-bit, winograd Schur K=64 "
                           "(alpha 2, n_min 32), A uniform [-1,1) full-mantissa (seed 11), b = A*1",
               "device_ms": float(np.mean(dev_ms)), "schur_leaf_ms": float(np.mean(leaf_ms)),
               "schur_leaf_madds": int(leaf_madds), "launches": int(launches),
               "schur_leaf_roofline": {"achieved": schur_tiops, "peak": leaf_peak_tiops, "unit": "TIOP/s (IMAD-eq)",
                                       "frac": schur_tiops / leaf_peak_tiops},
               "madd_per_s": (n ** 3 / 3) / (float(np.mean(dev_ms)) * 1e-3),
               "e2e": {"ms": e2e_ms, "api": "mpgpu_lu_blocked_host (the drop-in's lu_blocked: transfers overlapped with the factorisation), pinned host SoA, wall",
                       "h2d_bytes": nbytes_soa(n * n, L), "d2h_bytes": nbytes_soa(n * n, L)},
               "solve_ms": solve_ms, "solve": "column-oriented lu_solve (exact=False)",
               "forward_error_max_rel": fwd, "forward_error": "max_rel_error_solution(x, 1) in MP on the device"}
        for x_ in (work, src):
            x_.free()
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = lu_cpu_baseline(A, K, nmin)
        return out
    except Exception as e:  # reported, never fatal for the headline line
        return {"error": repr(e)[:300]}


def lu_cpu_baseline(A, K, nmin, s=256):
    """The compiled reference's lu_blocked (pivot-free: the reference has no pivoting) with the
    same Schur kernel, K and n_min on the top-left s x s block of the same A, one core,
    wall clock; extrapolated to n by the n^3 / 3 Schur work."""
    try:
        from oracle import oracle as O
        if not O.have_ref():
            return {"value": None, "sample": "oracle/_ref not built"}
        a = O.OMat.of(A.sub(0, 0, s, s))
        t0 = time.perf_counter()
        O.lu_blocked(a, K, "winograd", nmin, pivoting=False, which="ref")
        dt = time.perf_counter() - t0
        n = A.rows()
        return {"value": (s ** 3 / 3) / dt, "unit": "madd/s (n^3/3 per factorisation)", "cores": 1,
                "kind": "reference", "seconds_at_sample": dt,
                "extrapolated_seconds_at_n": dt * (n / s) ** 3,
                "sample": f"reference lu_blocked(winograd, K={K}, n_min={nmin}) pivot-free on the {s}x{s} top-left "
                          f"block of A, 1 core; n={n} time extrapolated by (n/{s})^3"}
    except Exception as e:
        return {"value": None, "sample": f"failed: {e}"}


def e2e(args, P, torch, a, b, algo, param, ctx, L):
    """Same metric through the reference-facing C-ABI call with HOST buffers
    (mpgpu_gemm_host): H2D of A, B from pinned memory, multiply, D2H of C."""
    def pinned_like(x):
        lim = torch.empty(x.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        ex = torch.empty(x.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
        sg = torch.empty(x.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
        return lim, ex, sg

    def pin(x):
        lim, ex, sg = pinned_like(x)
        lim[:] = x.limbs
        ex[:] = x.exp
        sg[:] = x.sign
        return P.Matrix(x.rows(), x.cols(), x.ctx(), lim, ex, sg)

    pa, pb = pin(a), pin(b)
    c = P.Matrix(a.rows(), b.cols(), ctx)
    lim, ex, sg = pinned_like(c)
    pc = P.Matrix(a.rows(), b.cols(), ctx, lim, ex, sg)
    P.gemm_host(algo, param, pa, pb, pc, ctx)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        P.gemm_host(algo, param, pa, pb, pc, ctx)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    n_el = a.rows() * a.cols()
    return {"value": a.rows() * a.cols() * b.cols() / dt, "unit": "madd/s",
            "h2d_bytes_per_step": nbytes_soa(n_el, pa.nlimbs) + nbytes_soa(b.rows() * b.cols(), pb.nlimbs),
            "d2h_bytes_per_step": nbytes_soa(a.rows() * b.cols(), pc.nlimbs), "ms_per_step": dt * 1e3,
            "api": "mpgpu_gemm_host (include/mpgpu.h), pinned host SoA buffers, wall clock around the call"}


def precision_sweep(args, P, torch, peak_tiops):
    """The north star's '>= 50 % of the IMAD roofline at 256-1024 bits': the same product
    (n, algorithm, n_min, full-mantissa inputs) at 256 / 512 / 1024 bits, leaf kernel only,
    CUDA-event timed (min of 3 after a warm-up).  Reported beside the headline line."""
    out = {}
    for bits in (256, 512, 1024):
        ctx = P.PrecisionContext(bits)
        n = args.n
        da = P.gen_uniform_full(n, n, 1, ctx).to_device()
        db = P.gen_uniform_full(n, n, 2, ctx).to_device()
        dc = P.DeviceMatrix(n, n, ctx)
        algo = P.Algorithm[args.algo]
        param = args.n_min if algo != P.Algorithm.simple else 0
        st = P.gemm_into(algo, param, da, db, dc)
        leaf = min(P.gemm_into(algo, param, da, db, dc).leaf_ms for _ in range(3))
        L = P.nlimbs_for(bits)
        achieved = st.leaf_madds * 2 * L * L / (leaf * 1e-3) / 1e12
        out[str(bits)] = {"leaf_ms": leaf, "leaf_madds": st.leaf_madds, "imad_eq_per_madd": 2 * L * L,
                          "achieved_tiops": achieved, "frac": achieved / peak_tiops,
                          "frac_issued": achieved / peak_tiops * issued_imad_eq_per_madd(L, bits) / (2 * L * L),
                          "device_ms_at_n_min": min(P.gemm_into(algo, param, da, db, dc).device_ms for _ in range(2))}
        if algo in (P.Algorithm.strassen, P.Algorithm.winograd):
            # the cutoff chosen per precision from the measured leaf throughput (MPGPU_AUTO_NMIN)
            nm, depth, model_ms = P.choose_n_min(algo, bits, n, n, n)
            P.gemm_into(algo, P.AUTO_NMIN, da, db, dc)
            auto = min((P.gemm_into(algo, P.AUTO_NMIN, da, db, dc) for _ in range(2)), key=lambda x: x.device_ms)
            out[str(bits)]["auto_n_min"] = {"n_min": nm, "depth": depth, "model_ms": model_ms,
                                            "device_ms": auto.device_ms, "leaf_ms": auto.leaf_ms}
        for x in (da, db, dc):
            x.free()
    torch.cuda.synchronize()
    return out


def owned_row_runs(runner, m: int, rank: int, world: int):
    """Contiguous runs [r0, r1) of the rows of C this rank reads back: its own rows for the
    row-owned and row-sharded runners, all of C for replicas, an even split otherwise."""
    from paper_1410_1599_b200 import shard
    if getattr(runner, "replicated", False):
        return [(0, m)]
    rows = getattr(runner, "c_rows", None)
    if rows is None:
        sh = getattr(runner, "shard", None) if runner.__class__.__name__ == "_RowSharded" else None
        sh = sh or shard.even_ranges(m, world)[rank]
        return [(sh.lo, min(sh.hi, m))] if sh.hi > sh.lo and sh.lo < m else []
    runs, start, prev = [], None, None
    for r in rows:
        if start is None:
            start = prev = r
        elif r == prev + 1:
            prev = r
        else:
            runs.append((start, prev + 1))
            start = prev = r
    if start is not None:
        runs.append((start, prev + 1))
    return runs


def e2e_dist(args, P, torch, dist, a, b, da, db, dc, runner, rank, world):
    """e2e at N > 1 through the public API on every rank: H2D of A and B from pinned host
    buffers (mpgpu_upload), the sharded product, D2H of the rows of C this rank owns
    (mpgpu_download of row views); wall clock per rank, max over ranks.  Every rank
    reaches the same collectives even if its upload / download fails."""
    import ctypes as C
    from paper_1410_1599_b200 import _lib as PL
    err, dt = None, float("inf")
    m, n = a.rows(), b.cols()
    runs = owned_row_runs(runner, m, rank, world)
    try:
        def pin(x):
            lim = torch.empty(x.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
            ex = torch.empty(x.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
            sg = torch.empty(x.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
            lim[:] = x.limbs
            ex[:] = x.exp
            sg[:] = x.sign
            return P.Matrix(x.rows(), x.cols(), x.ctx(), lim, ex, sg)

        pa, pb = pin(a), pin(b)
        outs = [P.Matrix(r1 - r0, n, a.ctx()) for r0, r1 in runs]
    except Exception as ex:
        err = repr(ex)[:300]

    def one(product=True):
        if err is None:
            da.upload(pa)
            db.upload(pb)
        if product:
            runner()  # collective: every rank calls it
        if err is None:
            for (r0, r1), o in zip(runs, outs):
                v = PL.MpgpuMat()
                PL.lib.mpgpu_matrix_view(C.byref(dc.m), r0, 0, r1 - r0, n, C.byref(v))
                rc = PL.lib.mpgpu_download(dc._h, C.byref(v), o.limbs.ctypes.data_as(C.c_void_p),
                                           o.exp.ctypes.data_as(C.c_void_p), o.sign.ctypes.data_as(C.c_void_p),
                                           o.nlimbs)
                if rc:
                    raise RuntimeError(f"mpgpu_download rc={rc}")

    try:
        one()
    except Exception as ex:
        err = err or repr(ex)[:300]
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        try:
            one()
        except Exception as ex:
            err = err or repr(ex)[:300]
    torch.cuda.synchronize()
    if err is None:
        dt = (time.perf_counter() - t0) / args.e2e_steps
    t = torch.tensor([dt], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    if err is not None or not np.isfinite(dt):
        return {"value": None, "unit": "madd/s", "error": err or "failed on another rank"}
    rows_read = sum(r1 - r0 for r0, r1 in runs)
    return {"value": m * a.cols() * n / dt, "unit": "madd/s",
            "h2d_bytes_per_step": nbytes_soa(m * a.cols(), a.nlimbs) + nbytes_soa(b.rows() * n, b.nlimbs),
            "d2h_bytes_per_step": nbytes_soa(rows_read * n, a.nlimbs), "ms_per_step": dt * 1e3,
            "api": "per rank: mpgpu_upload of A, B (pinned host SoA), the sharded product, mpgpu_download "
                   "of the rank's rows of C; bytes are rank 0's; wall clock, max over ranks"}


def cpu_baseline(args, P, a, b):
    """The compiled reference (oracle/_ref) on 1 host core, bounded sample."""
    try:
        from oracle import oracle as O
        if not O.have_ref():
            return {"value": None, "unit": "madd/s", "cores": 1, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        s, nmin_s = sample_shape(args)
        oa, ob = O.OMat.of(a.sub(0, 0, s, s)), O.OMat.of(b.sub(0, 0, s, s))
        reps, secs = 0, 0.0
        while secs < 10.0 and reps < 20:
            _, t = O.gemm_replicas(args.algo, nmin_s, oa, ob, 1)
            secs += t
            reps += 1
        return {"value": reps * s ** 3 / secs, "unit": "madd/s", "cores": 1, "kind": "reference",
                "sample": f"{reps} x " + sample_desc(args, s, nmin_s, 1)}
    except Exception as e:  # reported, never fatal
        return {"value": None, "unit": "madd/s", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}


if __name__ == "__main__":
    main()
