"""Benchmark: compressed NMF on BASELINE.json configs[1] (dense NMF, fp32,
m=10000, n=5000, r=20, two-sided compression with oversampling 10 and q=4,
then compressed ADMM for 500 iterations).

One "step" = the whole compressed-NMF job on device-resident A: both range
finders (2 x 9 streaming passes), the core L^T A R^T (one more pass), the
ADMM iterations and the final relative error (one more pass).

  value  = compression GB/s of A per pass: 19 passes x |A| / device time of
           the compression phase (BASELINE.json metric, first half);
  nmf_iters_per_s = ADMM iterations / device time of the ADMM phase (second
           half of the metric);
  e2e    = the same per-pass GB/s through the public API with host buffers:
           nmf_admm(pinned host A) -> host factors; 20 passes x |A| / wall
           time of the call (H2D of A, D2H of X, Y inside the timed region).

`--impl reference` times the CPU oracle port of the reference (numpy, all
host threads) on the same workload and reports the e2e-style number.
Multi-GPU (torchrun, N>1): A is sharded by columns (weak scaling: every
rank holds an m x 5000 shard of an m x 5000N matrix); the passes all-reduce
their m x S products over NCCL, CholeskyQR of row-sharded panels all-reduces
the S x S Gram matrix, the ADMM runs replicated on the compressed problem
(paper_1505_04650_b200/distributed.py); the time is the max over ranks.
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, N, R, R_OV, W, MAX_ITER, TOL, SEED = 10000, 5000, 20, 10, 4, 500, 1e-4, 5
PASSES_COMPRESS = 2 * (2 * W + 1) + 1   # two range finders + the core projection
PASSES_CALL = PASSES_COMPRESS + 1       # + relative-error pass
WORKLOAD = ("configs[1]: dense NMF fp32 m=10000 n=5000 r=20, X,Y~U[0,1], A=max(XY+N(0,0.01^2),0); "
            "two-sided compression r_ov=10 q=4; compressed ADMM 500 iterations")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_block(extra=None):
    c = {"workload": WORKLOAD, "m": M, "n": N, "r": R, "oversample": R_OV, "q": W, "admm_iters": MAX_ITER,
         "passes_compress": PASSES_COMPRESS, "l2": "inputs larger than L2 (A = 200 MB fp32 > 126 MB)",
         "parallelism": "A column-sharded across GPUs, m x 5000 per GPU (weak scaling)"}
    if extra:
        c.update(extra)
    return c


# --------------------------------------------------------------- oracle ----

def oracle_job(a):
    """The reference's CPU path (oracle port) for the same job."""
    from oracle import cnmf_oracle as O

    out = O.admm(a, R, compressed=True, cfg=O.Config(R, R_OV, W, SEED), max_iter=MAX_ITER, tol=TOL)
    return out


def synth_host(seed=0):
    import numpy as np

    g = np.random.default_rng(seed)
    x = g.uniform(size=(M, R)).astype(np.float32)
    y = g.uniform(size=(R, N)).astype(np.float32)
    a = x @ y + 0.01 * g.standard_normal((M, N), dtype=np.float32)
    return np.maximum(a, 0.0, out=a)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    a = synth_host().astype(np.float64)
    for _ in range(max(args.warmup, 1) if args.warmup else 0):
        oracle_job(a)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_job(a)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    gbs = PASSES_CALL * M * N * 4 / t / 1e9
    cores = os.cpu_count()
    line = {"metric": "compression GB/s of A per pass (% HBM roofline); compressed-NMF iters/sec",
            "value": gbs, "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_block({"reference_impl": "oracle port (numpy) of the reference cnmf package"}),
            "nmf_iters_per_s": MAX_ITER / t,
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
                             "sample": f"full configs[1] job, {args.steps} steps"},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours ----

class Clocks:
    """SM clock and throttle reasons sampled every 5 ms during the timed
    region (NVML in a background thread; nvidia-smi as the fallback)."""

    def __init__(self, index):
        import threading

        self.sm, self.mx, self.reasons, self.stop_ev = [], [], set(), threading.Event()
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nvml = None
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        if self.nvml is None:
            return
        n = self.nvml
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
        while not self.stop_ev.is_set():
            try:
                self.sm.append(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
                self.mx.append(n.nvmlDeviceGetMaxClockInfo(self.h, n.NVML_CLOCK_SM))
                fn = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    n.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for k, b in bits.items():
                    if r & b:
                        self.reasons.add(k)
            except Exception:
                pass
            self.stop_ev.wait(0.005)

    def stop(self):
        self.stop_ev.set()
        self.t.join()
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML every 5 ms during the timed steps"}


def run_ours(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1505_04650_b200 as C
    from paper_1505_04650_b200 import _lib
    from paper_1505_04650_b200.device import DeviceMatrix, stream, zeros
    from paper_1505_04650_b200.nmf import compressed_problem
    from paper_1505_04650_b200.rng import Rng

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()

    from paper_1505_04650_b200 import distributed as D

    # synthetic configs[1] data, generated on the device: X shared by all
    # ranks, this rank's column block Y_i and noise (global A = X [Y_0 .. Y_k])
    gx = torch.Generator(device="cuda").manual_seed(1234)
    g = torch.Generator(device="cuda").manual_seed(4321 + rank)
    x = torch.rand(M, R, device="cuda", generator=gx)
    y = torch.rand(R, N, device="cuda", generator=g)
    a = torch.addmm(0.01 * torch.randn(M, N, device="cuda", generator=g), x, y).clamp_(min=0.0)
    del x, y
    A = DeviceMatrix(a)
    n_glob, c0 = N * ws, N * rank
    cfg = C.adjust_config(C.CompressionConfig(r=R, r_ov=R_OV, w=W, seed=SEED), M, n_glob)
    comm, ops = D.Comm(), (D.DeviceOps() if ws > 1 else None)
    counts = [N] * ws
    s = cfg.basis_cols
    st = torch.cuda.current_stream()
    sp = stream()

    # buffers for the ADMM phase
    rng = Rng(cfg.seed)
    u0 = rng.child("init-left").uniform((M, R))
    vt0 = rng.child("init-right").uniform((R, n_glob), transpose=True)
    u, vt = u0.clone(), vt0.clone()
    du = zeros((M, R), torch.float64)
    dvt = zeros((n_glob, R), torch.float64)
    xc = zeros((s, R), torch.float64)
    yc = zeros((R, s), torch.float64)
    trace = zeros((MAX_ITER,), torch.float64)
    scores = zeros((MAX_ITER,), torch.float64)
    nbytes = lib.cnmf_admm_workspace(M, n_glob, s, R)
    wsb = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    it = ctypes.c_int(0)
    done = ctypes.c_int(0)
    res = zeros((2,), torch.float64)

    def step(ev):
        ev[0].record(st)
        if ws == 1:
            left, right, core = compressed_problem(A, cfg)
            lp, rp = left.panel, right.panel
        else:
            lp, right_local, core = D.compressed_problem(ops, comm, A, M, n_glob, c0, cfg)
            rp = comm.allgather_rows(right_local, counts)
        ev[1].record(st)
        u.copy_(u0)
        vt.copy_(vt0)
        _lib.call("cnmf_admm_run", core.data_ptr(), lp.data_ptr(), M, rp.data_ptr(), n_glob, s, R,
                  u.data_ptr(), du.data_ptr(), vt.data_ptr(), dvt.data_ptr(), xc.data_ptr(), yc.data_ptr(), 1.0, 1.0,
                  1.0, MAX_ITER, TOL, trace.data_ptr(), scores.data_ptr(), ctypes.byref(it), ctypes.byref(done), 0,
                  0, wsb.data_ptr(), nbytes, sp)
        ev[2].record(st)
        vloc = vt if ws == 1 else vt[c0: c0 + N].contiguous()
        _lib.call("cnmf_residual_norms", A.ptr, M, N, A.lda, u.data_ptr(), None, vloc.data_ptr(), R,
                  res.data_ptr(), sp)
        comm.allreduce(res)
        ev[3].record(st)
        return it.value

    for _ in range(args.warmup):
        step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()

    import paper_1505_04650_b200.nmf as nmf_mod

    clocks = Clocks(local)
    launches0 = lib.cnmf_launch_count() + nmf_mod.graph_launches
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(st)
    iters = [step(ev) for ev in evs]
    t_end.record(st)
    torch.cuda.synchronize()
    launches = lib.cnmf_launch_count() + nmf_mod.graph_launches - launches0
    ck = clocks.stop()
    # the dominant kernel timed live: one more compression, launched eagerly
    # (graph replays bypass the per-launch events), CUDA events around every
    # streaming pass on its launch stream
    lib.cnmf_set_pass_profiling(1)
    if ws == 1:
        compressed_problem(A, cfg, graph=False)
    else:
        D.compressed_problem(ops, comm, A, M, n_glob, c0, cfg)
    torch.cuda.synchronize()
    pms, pl, pby = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
    lib.cnmf_pass_stats(ctypes.byref(pms), ctypes.byref(pl), ctypes.byref(pby))
    lib.cnmf_set_pass_profiling(0)

    total_ms = t_start.elapsed_time(t_end)
    comp_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    admm_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    resid_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    t_local = torch.tensor([total_ms, comp_ms, admm_ms], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms, comp_ms, admm_ms = t_local.tolist()
    ms_per_step = total_ms / args.steps
    a_bytes = M * N * 4
    value = ws * PASSES_COMPRESS * a_bytes / (comp_ms * 1e-3) / 1e9
    iters_per_s = ws * (sum(iters) / len(iters)) / (admm_ms * 1e-3)

    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    pass_avg_ms = pms.value / max(pl.value, 1)
    pass_bytes = pby.value / max(pl.value, 1)
    achieved = pass_bytes / (pass_avg_ms * 1e-3) / 1e9
    sm_clock = (ck.get("sm_mhz") or 1965.0) * 1e6
    fp32_peak = 148 * 128 * 2 * sm_clock / 1e12  # FFMA peak at the observed SM clock
    pass_flops = 2.0 * M * N * 32  # padded panel width 32 for s = 30
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak,
                # dram__bytes_read.sum + dram__bytes_write.sum of one configs[1] pass_tc_pair launch (ncu --set
                # full, profiles/r01_pass_tc_pair_cfg1_ncu_full.txt): 332.88 MB + 6.72 MB against 403.8 MB
                # algorithmic -- the second direction's A tiles partly come from L2
                "traffic": 339.6e6 if (M, N) == (10000, 5000) else None, "traffic_unit": "bytes per paired launch",
                "algorithmic_bytes_per_launch": pass_bytes,
                "kernel": "pass_tc_pair<32> (both range finders' passes of a power step in one launch) + pass_tc<32> "
                          "(core projection), tcgen05 3xTF32, CUDA events on the launch stream",
                "launches": pl.value, "avg_launch_ms": pass_avg_ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                "fp32_tflops": pass_flops / (pass_avg_ms * 1e-3) / 1e12, "fp32_peak_tflops_at_clock": fp32_peak,
                "fp32_frac": pass_flops / (pass_avg_ms * 1e-3) / 1e12 / fp32_peak}

    # ---- end to end through the public API with host buffers ----
    a_host = a.cpu().pin_memory()
    cfg_pub = C.CompressionConfig(r=R, r_ov=R_OV, w=W, seed=SEED)

    def public_call():
        if ws == 1:
            fp = C.nmf_admm(a_host, R, cfg=cfg_pub, max_iter=MAX_ITER, tol=TOL)  # numpy out
            return fp.X.nbytes + fp.Y.nbytes + 8 * len(fp.objective_trace), fp.rel_error, fp.iterations
        uu, vv, it_, tr_, rel_ = D.nmf_admm(DeviceMatrix(a_host), M, n_glob, c0, R, cfg_pub, comm, ops,
                                            max_iter=MAX_ITER, tol=TOL)
        uh, vh = uu.cpu(), vv.cpu()
        return uh.numel() * 8 + vh.numel() * 8 + 8 * len(tr_), rel_, it_

    public_call()  # warm
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(1, min(args.steps, 3))):
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        d2h, rel_e2e, it_e2e = public_call()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    te_t = torch.tensor([sum(ts) / len(ts)], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
    te = te_t.item()
    e2e = {"value": ws * PASSES_CALL * a_bytes / te / 1e9, "unit": "GB/s", "h2d_bytes_per_step": a_bytes,
           "d2h_bytes_per_step": int(d2h), "ms": te * 1e3, "rel_error": rel_e2e, "iterations": it_e2e}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        a64 = a.cpu().double().numpy()
        t0 = time.perf_counter()
        oracle_job(a64)
        tc = time.perf_counter() - t0
        cpu = {"value": PASSES_CALL * a_bytes / tc / 1e9, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
               "sample": "one full configs[1] job (compression + 500 ADMM iterations + error) on the oracle port",
               "seconds": tc}

    if rank == 0:
        line = {"metric": "compression GB/s of A per pass (% HBM roofline); compressed-NMF iters/sec",
                "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "precision": "f32 passes over A; f64 Gram, Cholesky and ADMM state", "data": "synthetic",
                "config": config_block({"n_global": n_glob, "compress_ms": comp_ms, "admm_ms": admm_ms,
                                        "resid_ms": resid_ms,
                                        "hbm_frac_compress": value / ws / hbm_peak}),
                "nmf_iters_per_s": iters_per_s, "admm_iterations": iters[0],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": ck,
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
