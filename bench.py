"""bench.py — training throughput of the B200 PNN hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step is one pass of the whole hot path over the config's synthetic data:
E epochs of per-sample SGD of every CN on its slice, the
averaging merge incl. the cross-rank all-reduce (a7) and the test-set readout
of the merged network (a8).  value = Σ_ranks K_local·S·E / max_ranks(step time).
Scaling is strong: the config's K CNs and rows are split over the N ranks.

--impl reference times the CPU oracle (oracle/, the deliberately slow
single-threaded C trainer) on the host cores, on a bounded sample of the
same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS  # noqa: E402

METRIC = "training samples/sec (fwd+bwd+update, whole box)"


def fma_per_sample(layers):
    """Algorithmic FMAs per training sample: forward P,
    hidden deltas P - P1, update P  →  3P - P1 (P = weights, P1 = |W^1|)."""
    P = sum(layers[l] * layers[l - 1] for l in range(1, len(layers)))
    P1 = layers[0] * layers[1]
    return 3 * P - P1


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # noqa: BLE001
            self.error = str(e)
        return self

    def _run(self):
        nv = self._nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "n_samples": len(self.samples)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_sample(cfg, budget_s, cores=None):
    """Pick a bounded sample of the workload's CNs (≈budget_s of CPU work on
    `cores` host cores (default: all), ~1.2 GFLOP/s/core scalar fp32) and
    pre-generate its rows."""
    import oracle
    from datagen import make_rows
    oracle.build()
    cores = cores or len(os.sched_getaffinity(0))
    start, count = oracle.shard_bounds(cfg.n_train, cfg.K)
    S = int(count[0])
    per_cn = S * cfg.epochs * fma_per_sample(cfg.layers) * 2 / 1.0e9      # GFLOP per CN
    n_cn = int(max(1, min(cfg.K, budget_s * 1.2 * cores / per_cn)))
    if n_cn * per_cn > budget_s * 1.2 * cores:       # whole CNs overrun: one CN per core, fewer rows
        n_cn = min(cfg.K, cores)
        per_row = cfg.epochs * fma_per_sample(cfg.layers) * 2 / 1.0e9
        S = min(S, max(cfg.batch, int(budget_s * 1.2 / per_row) // cfg.batch * cfg.batch))
    if n_cn >= cores:
        n_cn = (n_cn // cores) * cores
    sample = list(range(n_cn))
    data = {int(start[i]): make_rows(int(start[i]), int(count[i]), "train", 0) for i in sample}
    if S < int(count[0]):                             # truncated slices (train on the first S rows)
        data = {k: (v[0][:S], v[1][:S]) for k, v in data.items()}
    threads = min(cores, n_cn)

    def run():
        oracle.train_pnn_rows(cfg.layers, cfg.act, cfg.init, cfg.K, cfg.lr, 0, cfg.n_train,
                              lambda s, c: data[s], epochs=cfg.epochs, batch=cfg.batch,
                              threads=threads, subnets=sample, precision=cfg.precision)

    desc = (f"{n_cn} of {cfg.K} CNs x {S} rows x {cfg.epochs} epoch(s), batch {cfg.batch}: "
            f"{cfg.precision} oracle, one CN per thread, {threads} threads; merge/readout not timed")
    return run, n_cn * S * cfg.epochs, threads, desc


def run_reference(args, cfg):
    """The oracle, as it stands, on the host cores (bounded sample per step)."""
    run, units, threads, desc = _oracle_sample(cfg, 4.0)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        run()
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    value = units / t
    return {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if cfg.precision == "fp32" else "bf16-emulated f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": cfg.name, "layers": list(cfg.layers), "K": cfg.K,
                   "rows": cfg.n_train, "epochs": cfg.epochs, "batch": cfg.batch},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "oracle",
                         "sample": desc, "cpu_model": cpu_model(), "host_cores": len(os.sched_getaffinity(0))},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline(cfg, budget_s=12.0):
    run, units, threads, desc = _oracle_sample(cfg, budget_s)
    t0 = time.perf_counter()
    run()
    t = time.perf_counter() - t0
    run1, units1, _, desc1 = _oracle_sample(cfg, 3.0, cores=1)      # the same oracle on one core
    t1 = time.perf_counter()
    run1()
    t1 = time.perf_counter() - t1
    return {"value": units / t, "unit": "samples/s", "cores": threads, "kind": "oracle",
            "sample": desc + f" ({t:.1f} s wall)", "cpu_model": cpu_model(),
            "host_cores": len(os.sched_getaffinity(0)), "single_core_value": units1 / t1,
            "single_core_sample": desc1 + f" ({t1:.1f} s wall)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "reference", "resident", "cluster"])
    ap.add_argument("--variant", default="auto",
                    choices=["auto", "v8", "v10", "tmem", "ws", "cluster", "deep", "mb_step", "mb_resident"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    import torch
    import torch.distributed as dist
    from datagen import make_rows
    from paper_2304_09590_b200 import PNN, PNN_BF16
    from paper_2304_09590_b200.dist import nccl_unique_id_bytes, rank_rows, rank_subnets

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")      # the driver counts the ranks in NCCL's log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    first, K_local = rank_subnets(cfg.K, world, rank)
    r0, nrows = rank_rows(cfg.n_train, cfg.K, world, rank)
    X, y = make_rows(r0, nrows, "train", 0)
    Xt, _ = make_rows(0, cfg.n_test, "test", 0)

    net = PNN(cfg.layers, cfg.act, cfg.init, cfg.K, cfg.lr, seed=0)
    net.set_kernel(args.kernel)
    if cfg.batch > 1:
        net.set_minibatch(cfg.batch, PNN_BF16 if cfg.precision == "bf16" else 0)
    if args.variant != "auto":
        net.set_variant(args.variant)
    if world > 1:
        net.set_comm(world, rank, nccl_unique_id_bytes(rank))
    kernel_id, launches_per_epoch = net.kernel_info()
    variant_id = net.kernel_variant()
    xd = torch.from_numpy(X).cuda()
    yd = torch.from_numpy(y).cuda()
    xtd = torch.from_numpy(Xt).cuda()
    labels = torch.empty(cfg.n_test, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(train_ev=None):
        for _ in range(cfg.epochs):
            if train_ev is not None:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            net.train_epoch(xd, yd, stream)
            if train_ev is not None:
                b.record(stream)
                train_ev.append((a, b))
        net.merge(stream)
        net.predict(xtd, labels, stream=stream)

    for _ in range(args.warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    train_ev = []
    net.kernel_timing(True)                   # CUDA events around each training-kernel launch
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step(train_ev)
        ev1.record(stream)
        barrier()
    kernel_ms, kernel_launches = net.kernel_timing(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    train_ms = statistics.mean(a.elapsed_time(b) for a, b in train_ev)
    t = torch.tensor([ms, train_ms, kernel_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, train_ms, kernel_ms = t.tolist()
    units = cfg.n_train * cfg.epochs          # all ranks together (strong scaling)
    value = units / (ms / 1e3)

    # ---- end to end through the host-buffer C-ABI call ----------------------
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(X).pin_memory()
        yh = torch.from_numpy(y).pin_memory()
        xth = torch.from_numpy(Xt).pin_memory()
        lab_h = torch.empty(cfg.n_test, dtype=torch.int32).pin_memory()

        if cfg.epochs > 1:                     # inputs copied once per step, then every epoch on them
            xe = torch.empty(X.shape, dtype=torch.float32, device="cuda")
            ye = torch.empty(y.shape, dtype=torch.int32, device="cuda")

        # The test rows go H2D on their own stream, after the previous step's readout released
        # xtd (an event, long complete by then): on the training stream the copy would queue
        # behind the training tail and stall the next step's input copies (C4: 69.3 vs 61.1 ms
        # per step, tools/e2e_probe.py).
        tcopy = torch.cuda.Stream()
        read_done = torch.cuda.Event()
        read_done.record(stream)

        def step_host():
            if cfg.epochs == 1:                # the host-buffer call pipelines H2D with training
                net.train_epoch_host(xh, yh, stream)
            else:
                with torch.cuda.stream(stream):
                    xe.copy_(xh, non_blocking=True)
                    ye.copy_(yh, non_blocking=True)
                for _ in range(cfg.epochs):
                    net.train_epoch(xe, ye, stream)
            net.merge(stream)
            tcopy.wait_event(read_done)
            with torch.cuda.stream(tcopy):
                xtd.copy_(xth, non_blocking=True)
            stream.wait_stream(tcopy)
            net.predict(xtd, labels, stream=stream)
            read_done.record(stream)
            with torch.cuda.stream(stream):
                lab_h.copy_(labels, non_blocking=True)

        for _ in range(max(1, args.warmup // 2)):
            step_host()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_host()
        e1.record(stream)
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": units / (ems.item() / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": int(X.nbytes + y.nbytes + Xt.nbytes),
               "d2h_bytes_per_step": int(lab_h.numel() * 4), "ms_per_step": ems.item()}

    if rank == 0:
        pk = peaks()
        clocks = clk.summary()
        sm_mhz = clocks["sm_mhz"] or pk.get("sm_max_mhz", 1965.0)
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        flop_launch = 2.0 * fma_per_sample(cfg.layers) * (nrows)   # this rank's launch
        # the dominant kernel's own launch duration (library CUDA events on this stream); the
        # epoch time (incl. the resident path's Gram pre-pass) is reported beside it
        kms = kernel_ms if kernel_launches else train_ms
        achieved = flop_launch / (kms / 1e3) / 1e12
        achieved_epoch = flop_launch / (train_ms / 1e3) / 1e12
        peak_max = sms * 128 * 2 * (pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        if cfg.precision == "bf16":
            # a10 is bound by the per-step fp32 master-weight update, not the tensor pipe:
            # per mini-batch step and CN, the GEMM layers' weights (W1, W2) are read and written
            # in fp32 (8 B), their bf16 copies written (W1b, W2b, W2bT: 2 B each) and read back by
            # the next step's GEMMs (2 B each)  [DESIGN.md §5]
            import math
            W1 = cfg.layers[0] * cfg.layers[1]
            W2 = cfg.layers[1] * cfg.layers[2]
            bytes_step = K_local * (8 * (W1 + W2) + 2 * 2 * (W1 + 2 * W2))
            steps_ep = math.ceil(math.ceil(nrows / K_local) / cfg.batch)
            gbs = bytes_step * steps_ep / (train_ms / 1e3) / 1e9
            hbm = pk.get("hbm_gbs", 6549.1)
            tflops_tc = achieved
            # The GEMMs are dense contractions on the tensor pipe: report against the sustained bf16
            # peak (the kernel sits inside a long step).  ncu shows small latency-bound grids with the
            # tensor pipe 2-11 % active and DRAM 12-17 % (profiles/r1f_ncu_summary.txt): the binding
            # resource is the per-step launch / dependency latency, not HBM; the modelled master-weight
            # bytes are reported beside it.
            peak_tc = pk.get("bf16_tflops_sustained", 1392.3)
            roof = {"bound": "tensor", "achieved": tflops_tc, "peak": peak_tc, "unit": "TFLOP/s",
                    "frac": tflops_tc / peak_tc, "traffic": None,
                    "kernel": "training epoch (bf16 mini-batch: weight cast + 7 launches per step, CUDA graph)",
                    "peak_note": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS, seconds-long loop); "
                                 "algorithmic flop = 2 x (3P - P1) per sample; latency-bound per ncu",
                    "modelled_hbm": {"achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
                                     "bytes_per_step": bytes_step,
                                     "model": "K_local x (8(W1+W2) + 4(W1+2 W2)) per mini-batch step"},
                    "train_ms_per_launch": train_ms, "flop_per_launch": flop_launch}
        else:
            traffic = None
            ncu_extra = None
            try:      # dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel, per launch,
                      # from the committed ncu --set full capture of this workload
                tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(
                    f"{cfg.name}/{variant_id}")
                if tr and K_local == cfg.K and kernel_id in (2, 5):
                    traffic = tr["bytes_per_launch"]
                    ncu_extra = {k: tr[k] for k in ("fma_pipe_active_pct", "issue_active_pct", "smem_tbs",
                                                    "smem_peak_tbs", "smem_frac", "note", "source") if k in tr}
            except Exception:  # noqa: BLE001
                traffic = None
            roof = {"bound": "alu", "achieved": achieved, "peak": peak_max,
                    "unit": "TFLOP/s", "frac": achieved / peak_max, "traffic": traffic,
                    "traffic_note": "bytes/launch (ncu capture, profiles/ncu_traffic.json); algorithmic: "
                                    "X 4·784·rows + 2·4·P_total·K (+ 32-B Gram records·rows on the v8 / deep "
                                    "paths, whose Gram pre-pass is a separate launch)",
                    "kernel": {1: "training epoch (reference kernel)",
                               2: ("persistent SGD launch, TMEM variant (k_tmem.cu: one SM per CN, W1 in "
                                   "registers + tensor memory, Gram terms formed in the launch)"
                                   if variant_id == 11 else
                                   "persistent SGD launch, warp-specialised TMEM variant (k_ws.cu: one SM per CN, "
                                   "W1 in registers + tensor memory + shared memory, paired sweeps on 8 warps, the "
                                   "per-sample chain on its own warpgroup; frac_epoch adds the Gram pre-pass)"
                                   if variant_id == 12 else
                                   "persistent SGD launch (library CUDA events around it; frac_epoch adds the "
                                   "Gram pre-pass)"),
                               5: ("training epoch (deep cluster variant: Gram pre-pass + W1 in the registers and "
                                   "tensor memory of a 4-CTA cluster, k_deep.cu)" if launches_per_epoch == 2 else
                                   "training epoch (cluster kernel, weights in cluster shared memory)"),
                               4: "training epoch (fp32 mini-batch: 4 launches per step, CUDA graph)",
                               6: "training epoch (fp32 mini-batch, one persistent launch: W1 register-resident "
                                  "over a cluster, k_mbres.cu)"}
                              .get(kernel_id, "training epoch"),
                    "peak_note": f"FP32 FMA: {sms} SMs x 128 FMA/clk x 2 flop x "
                                 f"{pk.get('sm_max_mhz', 1965.0):.0f} MHz (guide unit counts, "
                                 f"sm_max clock); at the measured {sm_mhz:.0f} MHz the frac "
                                 f"is {achieved / (peak_max * sm_mhz / pk.get('sm_max_mhz', 1965.0)):.3f}",
                    "kernel_ms_per_launch": kms, "train_ms_per_epoch": train_ms,
                    "frac_epoch": achieved_epoch / peak_max,
                    "flop_per_launch": flop_launch}
            if ncu_extra:
                roof["ncu"] = ncu_extra
        import math
        steps_epoch = math.ceil(math.ceil(nrows / K_local) / cfg.batch)
        if kernel_id == 3:          # bf16 tcgen05 mini-batch: weight cast + 7 per step
            launches_epoch = 1 + launches_per_epoch * steps_epoch
        elif kernel_id == 4:        # fp32 mini-batch step kernels: 4 per step
            launches_epoch = launches_per_epoch * steps_epoch
        else:
            launches_epoch = launches_per_epoch
        out = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if cfg.precision == "bf16" else "f32",
            "data": "synthetic (seeded MNIST-shaped stand-in, datagen/)",
            "config": {"workload": f"{cfg.name}: {'-'.join(map(str, cfg.layers))} "
                                   f"{'/'.join(cfg.act)}, {cfg.init} init, K={cfg.K} CNs, "
                                   f"{cfg.n_train} rows, {cfg.epochs} epoch(s), batch {cfg.batch}, "
                                   f"lr {cfg.lr}",
                       "K_local": K_local, "rows_per_rank": nrows, "test_rows": cfg.n_test,
                       "kernel": ["auto", "reference", "resident", "tc_bf16", "mb_f32", "cluster", "mb_resident"][kernel_id],
                       "variant": {0: "none", 8: "v8", 10: "v10", 11: "tmem", 12: "ws", 20: "cluster", 21: "deep",
                                   30: "mb_step", 31: "mb_resident"}.get(variant_id, str(variant_id)),
                       "l2": f"inputs {X.nbytes / 2**20:.0f} MiB per rank > 126 MB L2 (no flush)"},
            "roofline": roof,
            "breakdown_ms": {"train": train_ms * cfg.epochs, "merge_predict": ms - train_ms * cfg.epochs},
            "clocks": clocks,
            "gpu_launches": args.steps * (cfg.epochs * launches_epoch + 2),
        }
        if e2e:
            out["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    net.close()


if __name__ == "__main__":
    main()
