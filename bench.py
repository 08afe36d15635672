#!/usr/bin/env python
"""bench.py — wedges/s and balanced butterflies/s of the B200 path (BASELINE.json `metric`).

One step = the whole hot path over one synthetic graph already resident in HBM: load the
signed CSR from device memory (validate, degrees, priority ranks, rank-space adjacency, work
plan: S1-S5), count global + per-vertex balanced/unbalanced butterflies (S6-S9), and, with
N > 1 GPUs, the NCCL all-reduce of the per-vertex arrays (S12); then free the graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Multi-GPU: launch with torchrun (one process per GPU); the graph is replicated, start-vertex
work units are sharded across ranks, and the library all-reduces the counts.
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

METRIC = "wedges/sec and balanced butterflies/sec at 1/2/4/8 B200; % HBM roofline"
WORKLOADS = {
    1: "configs[0]: uniform 200x150, 2,000 edges, p+=0.7",
    2: "configs[1]: actor-movie 5,000x4,800, ~24K edges, per-movie signs",
    3: "configs[2]: Chung-Lu 1M x 200K, 10M edges, gamma=2.1, p+=0.8",
    4: "configs[3]: dense block 16,384^2, density 0.05, p+=0.5",
    5: "configs[4]: Chung-Lu 8M x 2M, 50M edges, gamma=1.9, per-V Beta(3,1) sign bias",
    6: "NEXT-3 hybrid workload (not a BASELINE config): 8,192^2 community at density 0.2 in a Chung-Lu "
       "1M x 200K periphery (5M edges, gamma=2.1, weight max 1,000), p+=0.8",
}


def peaks():
    """(HBM GB/s, source), (int8 dense TOP/s, source).  int8 is not in MEASURED_PEAKS.json: it is
    the measured bf16 burst figure x 2, the guide's nominal int8 (4.5 POPS) / bf16 (2.25 PF) ratio."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        hbm = (float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)")
        i8 = (2.0 * float(p["bf16_tflops"]),
              "MEASURED_PEAKS.json bf16_tflops (burst) x 2 (nominal int8/bf16 ratio 4.5/2.25)")
    except Exception:
        hbm = (6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)")
        i8 = (4500.0, "nominal B200 dense int8 4.5 POPS (no measured peak available)")
    return hbm, i8


def measured_tensor_peaks():
    """Library GEMM peaks measured on this pool (tools/microbench/fp4_peak.py ->
    profiles/r2_microbench_peaks.jsonl, best of 10 at 8192^3): FP4 block-scaled and int8, TOP/s."""
    out = {}
    try:
        for line in open(os.path.join(ROOT, "profiles", "r2_microbench_peaks.jsonl")):
            r = json.loads(line)
            if r.get("n") != 8192:
                continue
            if r["bench"] == "fp4_block_scaled_mm":
                out["fp4"] = r["tflops"]
            elif r["bench"] == "int8_int_mm":
                out["int8"] = r["tops"]
    except OSError:
        pass
    return out


def ncu_tensor_util(kernel: str):
    """Tensor-pipe utilisation of `kernel` from its committed ncu capture summary
    (profiles/r2_ncu_dense_tensor_pipe.json: sm__pipe_tensor_cycles_active, % of peak elapsed)."""
    try:
        for r in json.load(open(os.path.join(ROOT, "profiles", "r2_ncu_dense_tensor_pipe.json"))):
            if kernel in r["kernel"]:
                return float(r["metrics"]["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]) / 100
    except (OSError, KeyError, ValueError):
        pass
    return None


def hybrid_evidence():
    """The hybrid path's fused cross-term kernel (k_dense_f4q<true>) from its committed ncu --set
    full summary (profiles/r2_ncu_k_dense_f4q_cross_c6.json): time and tensor-pipe utilisation."""
    try:
        r = json.load(open(os.path.join(ROOT, "profiles", "r2_ncu_k_dense_f4q_cross_c6.json")))[0]["metrics"]
        return {"kernel": "k_dense_f4q<true> (fused cross terms of the mixed core pairs, tcgen05 kind::mxf4)",
                "us_per_launch_ncu": float(r["gpu__time_duration.sum"][0]),
                "tensor_pipe_util_ncu": float(r["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]) / 100,
                "source": "profiles/r2_ncu_k_dense_f4q_cross_c6.json (config 6)"}
    except (OSError, KeyError, ValueError, IndexError):
        return None


def ncu_traffic(config: int, kernel: str):
    """dram read+write bytes per launch of `kernel` on `config` from the committed ncu --set full
    summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{kernel}@{config}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def expected_counts(config: int):
    """The oracle's counts for `config` (tests/golden/expected_counts.json, written by
    tests/scripts/write_expected.py, which calls only oracle/)."""
    with open(os.path.join(ROOT, "tests", "golden", "expected_counts.json")) as f:
        return json.load(f)[f"config{config}"]


def pv_sha256(arrays) -> str:
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype="<u8").tobytes())
    return h.hexdigest()


def check_parity(g, config: int, tot: dict, pv) -> dict:
    """Bit-exact parity gate run before any throughput number is printed: B, N, W_G and the
    per-vertex arrays of this run against the oracle's expected-counts file.  Raises on a
    mismatch."""
    exp = expected_counts(config)
    assert exp["graph_sha256"] == g.sha256(), "synthetic graph differs from the one the oracle counted"
    got = (tot["balanced"], tot["unbalanced"], tot["wedges_G"])
    want = (exp["B"], exp["N"], exp["W_G"])
    assert got == want, f"parity: (B, N, W_G) {got} != oracle {want}"
    sha = pv_sha256(pv)
    assert sha == exp["pv_sha256"], "parity: per-vertex arrays differ from the oracle's"
    return {"B": exp["B"], "N": exp["N"], "W_G": exp["W_G"], "pv_sha256": sha,
            "graph_sha256": exp["graph_sha256"],
            "source": "tests/golden/expected_counts.json (oracle_route_g_pv)"}


def cpu_baseline(g, pv=None, single_thread_configs=(1, 2, 3)):
    """The oracle as it stands (oracle/bbf_oracle.c oracle_route_g_pv: Alg. 2 / ParBB-Bucket with
    the 4-role scatter, dynamic chunks of 4 starts over all host threads) on the WHOLE graph — global
    and per-vertex counts, the same outputs as the GPU step.  value = W_G / its counting-loop time.
    When `pv` (the GPU's per-vertex arrays) is given, they are compared with the oracle's element
    by element in this same run (raises on a mismatch).  Also the single-thread Alg. 2 time
    (global counts) of the small configs, as the paper reports sequential BB-Bucket."""
    import oracle as O
    from synth import graphs as G
    threads = os.cpu_count() or 1
    r = O.route_g_pv(g, threads=threads)
    if pv is not None:
        for name, a in zip(("bal_u", "unb_u", "bal_v", "unb_v"), pv):
            assert np.array_equal(np.asarray(a).view(np.uint64), r[name]), f"parity vs oracle: {name}"
    single = {}
    for c in single_thread_configs:
        s = O.route_g(G.make_config(c), threads=1)
        single[f"config{c}"] = {"seconds": s["count_s"], "wedges_G": s["W_G"],
                                "wedges_per_s": s["W_G"] / max(s["count_s"], 1e-9)}
    return {"value": r["W_G"] / max(r["count_s"], 1e-9), "unit": "wedges/s", "cores": threads,
            "kind": "oracle", "cpu_model": cpu_model(),
            "sample": (f"the whole workload: oracle_route_g_pv (Alg. 2 + 4-role scatter, global + "
                       f"per-vertex counts) over all {g.n_u + g.n_v} start vertices, "
                       f"{r['W_G']:.4e} wedges, counting loop {r['count_s']:.2f} s on {threads} threads "
                       f"(graph build and adjacency sort excluded)"),
            "seconds": r["count_s"], "wedges": r["W_G"],
            "parity_vs_gpu_arrays": pv is not None,
            "single_thread_route_g_global": single}


def reference_arm(args):
    """--impl reference: the CPU oracle as it stands (oracle_route_g_pv, all host threads), on this
    arm's config/metric.  Step i counts start slice i of W+K deterministic disjoint slices (start x
    in slice x mod (W+K)), so the whole run is one full pass over the graph and every timed step is
    a bounded, reproducible sample of it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    from synth import graphs as G
    g = G.make_config(args.config)
    threads = os.cpu_count() or 1
    S = args.warmup + args.steps
    ids = np.arange(g.n_u + g.n_v, dtype=np.uint32)
    W = T = 0.0
    with O.Prepared(g) as h:  # Alg. 2 lines 2-3 once; each step times the counting loop
        for i in range(S):
            r = h.route_g_pv(starts=ids[i::S], threads=threads)
            if i >= args.warmup:
                W += r["W_G"]
                T += r["count_s"]
    v = W / max(T, 1e-9)
    sample = (f"oracle_route_g_pv (Alg. 2 + 4-role scatter, global + per-vertex) on {threads} threads; "
              f"step = start slice (x mod {S}); the {args.steps} timed slices hold {W:.4e} wedges")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "wedges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * T / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "uint32+uint128", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "counts": "global + per-vertex (both sides)"},
            "cpu_baseline": {"value": v, "unit": "wedges/s", "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": v, "unit": "wedges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=-1, help="e2e timed steps (default: --steps)")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampler")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    from paper_2308_07932_b200 import bbf
    from synth import graphs as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        from paper_2308_07932_b200 import dist as D
        dist.init_process_group("nccl", device_id=dev)
        comm = D.make_comm(local)  # the library's own NCCL communicator (id broadcast over torch)

    g = G.make_config(args.config)
    n_u, n_v = g.n_u, g.n_v
    rp = torch.from_numpy(g.row_ptr.view(np.int64)).to(dev)
    col = torch.from_numpy(g.col.view(np.int32)).to(dev)
    sg = torch.from_numpy(g.sign).to(dev)
    outs = tuple(torch.zeros(k, dtype=torch.int64, device=dev) for k in (n_u, n_u, n_v, n_v))
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def step():
        h = bbf.Graph(n_u, n_v, rp, col, sg, device=local, stream=stream, comm=comm)
        tot = h.count_per_vertex(out=outs)[0]
        st = h.stats()
        st["hybrid_core"] = h.hybrid_core()
        h.free()
        return tot, st

    for _ in range(args.warmup):
        tot, st = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    if not args.no_clocks:
        clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    main_ms = []
    count_ms = []
    algo_bytes = 0
    algo_ops = 0.0
    e0.record(stream)
    for _ in range(args.steps):
        tot, st = step()
        launches += st["kernel_launches"]
        main_ms.append(st["ms_main_kernel"])
        count_ms.append(tot["ms_count"])
        algo_bytes = st["algo_bytes"]
        algo_ops = st["algo_ops"]
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    W_G = tot["wedges_G"]
    cms = float(np.mean(count_ms))
    if world > 1:
        t = torch.tensor([cms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        cms = float(t.item())
    value = W_G * args.steps / (ms * 1e-3)
    bfly = tot["balanced"] * args.steps / (ms * 1e-3)
    # parity gate (bit-exact, before anything is printed): the last timed step's counts and
    # per-vertex arrays against the oracle's
    pv_host = [o.cpu().numpy().view(np.uint64) for o in outs]
    parity = check_parity(g, args.config, tot, pv_host)

    # e2e: the same step through the public API with HOST buffers, pipelined as a stream of
    # graphs: every step's CSR is copied from pinned host memory by bbf_upload_csr (the next
    # step's copy is started before this step counts, so it overlaps the kernels) and every
    # step's per-vertex arrays are written back to pinned host memory by BBF_OUTPUT_ASYNC copies
    # (overlapping the next step); all copies of all steps lie inside the timed region, which
    # ends after bbf_device_sync
    e2e_ms = None
    if args.e2e_steps < 0:
        args.e2e_steps = args.steps
    if args.e2e_steps > 0:
        h_rp = torch.from_numpy(g.row_ptr.view(np.int64)).pin_memory()
        h_col = torch.from_numpy(g.col.view(np.int32)).pin_memory()
        h_sg = torch.from_numpy(g.sign).pin_memory()
        h_out = tuple(torch.zeros(k, dtype=torch.int64).pin_memory() for k in (n_u, n_u, n_v, n_v))
        up = bbf.Upload(n_u, n_v, h_rp, h_col, h_sg, device=local)  # warm-up: the same pipelined loop
        for k in range(max(args.warmup, 1)):
            h = bbf.Graph.from_upload(up, stream=stream, comm=comm)
            if k + 1 < max(args.warmup, 1):
                up = bbf.Upload(n_u, n_v, h_rp, h_col, h_sg, device=local)
            h.count_per_vertex(out=h_out, flags=bbf.BBF_OUTPUT_ASYNC)
            h.free()
        bbf.device_sync(local)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        up = bbf.Upload(n_u, n_v, h_rp, h_col, h_sg, device=local)
        for k in range(args.e2e_steps):
            h = bbf.Graph.from_upload(up, stream=stream, comm=comm)
            if k + 1 < args.e2e_steps:
                up = bbf.Upload(n_u, n_v, h_rp, h_col, h_sg, device=local)
            tot_e = h.count_per_vertex(out=h_out, flags=bbf.BBF_OUTPUT_ASYNC)[0]
            h.free()
        bbf.device_sync(local)
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = t0.elapsed_time(t1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        assert tot_e["balanced"] == tot["balanced"]
        # the host-buffer path's outputs pass the same parity gate
        assert pv_sha256([o.numpy().view(np.uint64) for o in h_out]) == parity["pv_sha256"]
    h2d = g.row_ptr.nbytes + g.col.nbytes + g.sign.nbytes
    d2h = 8 * 2 * (n_u + n_v)

    (hbm_peak, hbm_src), (i8_peak, i8_src) = peaks()
    kms = float(np.mean(main_ms)) if main_ms else 0.0
    # the dense path runs on the block-scaled FP4 tensor cores when the rows' max degree keeps
    # the fp32 accumulation exact (<= 8192, csrc/dense_i8.cu), else on the int8 ones
    maxdeg = int(max(np.diff(g.row_ptr.astype(np.int64)).max(initial=0),
                     np.bincount(g.col, minlength=1).max(initial=0)))
    f4 = maxdeg <= 8192 and not os.environ.get("BBF_DENSE_I8")
    if algo_ops > 0 and f4:
        achieved = algo_ops / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
        f4_peak = 2.0 * i8_peak  # measured bf16 burst x 4 (nominal fp4 / bf16 = 9 / 2.25)
        kname = ("k_dense_f4q (tcgen05.mma.cta_group::2 kind::mxf4, e2m1 operands, one accumulator "
                 "Q = T + 2048 P via block scales, double-buffered TMEM)" if maxdeg < 2048 and
                 not os.environ.get("BBF_DENSE_F4_TP") else
                 "k_dense_f4 (tcgen05.mma.cta_group::2 kind::mxf4, e2m1 operands, T=AA^T and P=SS^T)")
        roof = {"bound": "tensor",
                "kernel": kname,
                "achieved": achieved, "peak": f4_peak,
                "peak_source": i8_src.replace("x 2 (nominal int8/bf16 ratio 4.5/2.25)", "x 4 (nominal fp4/bf16 ratio 9/2.25)"),
                "unit": "TOP/s (fp4, ops = 2 per MAC of the exact integer products)",
                "frac": achieved / f4_peak, "traffic": ncu_traffic(args.config, kname.split()[0]),
                "nominal_peak": 9000.0, "frac_of_nominal": achieved / 9000.0,
                "measured_library_peak": measured_tensor_peaks().get("fp4"),
                "measured_library_peak_source": "cuBLASLt FP4 block-scaled GEMM via torch._scaled_mm, 8192^3 best of 10 "
                                                "(profiles/r2_microbench_peaks.jsonl); the kernel exceeds it",
                "tensor_pipe_util_ncu": ncu_tensor_util(kname.split()[0]),
                "algo_ops_per_launch": algo_ops, "kernels_per_step": 2}
    elif algo_ops > 0:  # dense int8 tensor-core path (k_dense_pair)
        achieved = algo_ops / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
        roof = {"bound": "tensor",
                "kernel": "k_dense_pair (tcgen05.mma.cta_group::2 kind::i8, T=AA^T and P=SS^T)",
                "achieved": achieved, "peak": i8_peak, "peak_source": i8_src, "unit": "TOP/s (int8)",
                "frac": achieved / i8_peak, "traffic": ncu_traffic(args.config, "k_dense_pair"),
                "nominal_peak": 4500.0, "frac_of_nominal": achieved / 4500.0,
                "measured_library_peak": measured_tensor_peaks().get("int8"),
                "tensor_pipe_util_ncu": ncu_tensor_util("k_dense_pair"),
                "note": "int8 has no measured peak on this pool; the derived one (bf16 burst x 2) is "
                        "below what the kernel reaches (cuBLASLt int8 8192^3 measured 3322 TOP/s, "
                        "profiles/r1_microbench_int8_bf16_hbm.jsonl)",
                "algo_ops_per_launch": algo_ops, "kernels_per_step": 2}
    else:  # sparse path, hub wedge-aggregation kernel
        achieved = algo_bytes / (kms * 1e-3) / 1e9 if kms > 0 else 0.0
        roof = {"bound": "hbm", "kernel": "k_t3 (hub wedge aggregation)",
                "achieved": achieved, "peak": hbm_peak, "peak_source": hbm_src, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": ncu_traffic(args.config, "k_t3"),
                "algo_bytes_per_launch": algo_bytes}
    roof.update({"ms_per_launch": kms, "share_of_step": kms / ms_step if ms_step else None})
    dtype = ("e2m1 x e2m1 -> fp32 (exact integers) + uint64" if algo_ops > 0 and f4 else
             "int8 x int8 -> int32 + uint64" if algo_ops > 0 else "uint32 + uint64")

    line = {
        "metric": METRIC, "value": value, "unit": "wedges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "counts": "global + per-vertex (both sides)",
                   "path": ("hybrid dense core %d x %d + sparse remainder (DESIGN.md §6b)" % st["hybrid_core"]
                            if st["hybrid_core"] != (0, 0) else "dense" if algo_ops > 0 else "sparse"),
                   "wedges_G": W_G, "balanced": tot["balanced"], "unbalanced": tot["unbalanced"],
                   "step": "bbf_graph_load_csr(device CSR) + bbf_count_per_vertex + free",
                   "l2": f"inputs larger than L2 (input CSR {(g.row_ptr.nbytes + g.col.nbytes + g.sign.nbytes) / 1e6:.0f} MB "
                         f"+ rank-space CSR + build buffers > 126 MB); no flush",
                   "parallelism": f"dp{world} (start-vertex units sharded, CSR replicated)"},
        "balanced_butterflies_per_s": bfly,
        # SURVEY §8(d)'s t_count reading: graph already resident and built, the count call alone
        # (plan + wedge kernels + NCCL all-reduce; bbf_counts.ms_count)
        "count_only": {"value": W_G / (cms * 1e-3) if cms > 0 else None, "unit": "wedges/s",
                       "ms_per_step": cms, "definition": "W_G / device time of the count inside "
                       "bbf_count_per_vertex (plan + kernels + all-reduce); load/build excluded"},
        "e2e": {"value": (W_G / (e2e_ms * 1e-3)) if e2e_ms else None, "unit": "wedges/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms,
                "mode": "stream of graphs: bbf_upload_csr (pinned H2D) of step k+1 overlaps step k, "
                        "per-vertex arrays D2H by BBF_OUTPUT_ASYNC; all copies inside the timed region"},
        "gpu_launches": launches,
        "roofline": roof,
        "clocks": clocks,
    }
    line["parity"] = parity
    if st["hybrid_core"] != (0, 0):
        line["hybrid"] = {"core": list(st["hybrid_core"]), "fused_cross_kernel": hybrid_evidence(),
                          "note": "roofline above = the engine's hub kernel on the sparse remainder; the dense "
                                  "core and cross terms run on the FP4 tensor cores (DESIGN.md §6b)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(g, pv=pv_host)
        line["cpu_baseline"].pop("wedges", None)
        line["parity"]["oracle_run_in_this_job"] = True
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm:
        comm.free()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
