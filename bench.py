#!/usr/bin/env python
"""Benchmark of the FD-CNN DPD downlink hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one pass of the whole hot path over one batch
of synthetic OFDM symbols.  Default workload: BASELINE.json configs[4] = C5, the
north-star configuration (U=32, B=512, N_ifft=16384, N_d=3300, 256-QAM, 5-layer 64-channel
FD-CNN), 32 symbols per GPU per step (SURVEY §8(d) streaming batch; the 4096-symbol run's
275 GB waveform never coexists in memory).  Step: FD-CNN -> precode -> fused IDFT/GMP (PA
waveform written to HBM) + receive DFT -> channel sum + slicing/SER.  The ZF precoder (a2)
is built once per channel realisation before timing (reading A10) and timed separately.

Multi-GPU (torchrun): symbol-batch sharding (Mode S), weak scaling — each rank runs its
own batch (symbol indices rank*n + i); the only collective is the int64 SER-counter
all-reduce of each step.  Timing: CUDA events per step on the launching stream, L2
flushed between steps (256 MiB write, outside the events), barrier + synchronize around
the timed loop, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workload import configs, gen  # noqa: E402

METRIC = "OFDM symbols/s through DPD+precode+IFFT+GMP chain; % HBM roofline"
FP32_LANES_PER_SM = 128          # FP32 FMA lanes per SM (Blackwell SM: 4 SMSP x 32)


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-measured on this pool's B200s), else the
    fallback of /opt/skills/guides/B200_PROFILING.md (6.65 TB/s, 1.59 PFLOP/s bf16)."""
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m.get(k, p[k]) for k in ("hbm_gbs", "bf16_tflops", "sm_max_mhz")}, src="measured")
    return p


def gmp_flop_per_sample(cfg):
    """3 (envelope) + (Kp-2) (powers) + (L+1)[4(Kp-1)(2M+1) + 8]."""
    return 3 + (cfg.Kp - 2) + (cfg.L + 1) * (4 * (cfg.Kp - 1) * (2 * cfg.M + 1) + 8)


def chain_tx_flop_per_symbol(cfg):
    """Algorithmic FLOPs of the fused precode + IDFT + GMP per OFDM symbol."""
    N = cfg.N_ifft
    return (8 * cfg.B * cfg.U * cfg.N_d                       # precode, Eq. (1)
            + 5 * N * int(np.log2(N)) * cfg.B                  # IDFT, 5 N log2 N (P:165 convention)
            + gmp_flop_per_sample(cfg) * N * cfg.B)            # GMP, Eq. (9)


def chain_bytes_per_symbol(cfg, fused=True):
    """Algorithmic HBM bytes of the step per symbol: read s and idx, write the PA waveform y
    once (plus read it back when the receive is not fused), write yhat; P and h_fd amortised
    over the batch."""
    s = 8 * cfg.U * cfg.N_d
    y = 8 * cfg.B * cfg.N_ifft
    return s + 2 * cfg.U * cfg.N_d + (1 if fused else 2) * y + s + (16 * cfg.B * cfg.U * cfg.N_d) / cfg.n_sym


def measured_traffic(cfg, n, args):
    """DRAM bytes per chain_txrx launch from the committed ncu --set full capture of this exact
    launch configuration (profiles/traffic_<cfg>.json), else None."""
    path = os.path.join(ROOT, "profiles", f"traffic_{cfg.name.lower()}.json")
    if args.unfused or args.impair or args.redraw or not os.path.exists(path):
        return None
    with open(path) as f:
        t = json.load(f).get("chain_txrx")
    return t["bytes_per_launch"] if t and t.get("batch") == n else None


# ============================================================================ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 200.0] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "power_w_max": max(r[2] for r in rows)}


# ============================================================================ oracle timing
def git_sha():
    """The commit, or (on a GPU box, where the snapshot has no .git) a sha256 over the product
    sources and bench.py, so a line can be matched to the code that produced it."""
    try:
        sha = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], cwd=ROOT, capture_output=True, text=True,
                             timeout=10).stdout.strip()
        if sha:
            return sha
    except Exception:
        pass
    import hashlib
    h = hashlib.sha256()
    for d in ("paper_2205_05158_b200/csrc", "include", "paper_2205_05158_b200"):
        full = os.path.join(ROOT, d)
        for f in sorted(os.listdir(full)):
            if f.endswith((".cu", ".cuh", ".h", ".py")):
                with open(os.path.join(full, f), "rb") as fh:
                    h.update(fh.read())
    with open(os.path.join(ROOT, "bench.py"), "rb") as fh:
        h.update(fh.read())
    return "src-" + h.hexdigest()[:16]


def oracle_sample(cfg, first_symbol, budget_cpu_s=20.0, max_wall_s=60.0, workers=None):
    """Time the fp64 oracle (as it stands, oracle/parallel.py) on a bounded sample of the workload:
    per-step stages (CNN, precode, IDFT, GMP, receive, slice) one OFDM symbol at a time, spread over
    all host cores; ZF built untimed like the GPU's.  Runs symbols until ~budget_cpu_s of CPU work
    (at least one).  Returns the cpu_baseline dict."""
    from oracle import parallel as OP
    cores = OP.host_cores() if workers is None else workers
    per_sym_guess = {"C1": 0.002, "C2": 0.35, "C3": 1.7, "C4": 18.0, "C5": 45.0}.get(cfg.name[:2], 1.0)
    k = int(max(1, min(64, budget_cpu_s // per_sym_guess)))
    symbols = list(range(first_symbol, first_symbol + k))
    inp = gen.make_inputs(cfg, symbols)
    walls, cpus = [], []
    with OP.OracleRunner(cfg, inp, workers=cores) as r:
        for i in range(k):
            _, w, c = r.symbol(i)
            walls.append(w)
            cpus.append(c)
            if sum(walls) > max_wall_s:
                break
    n = len(walls)
    return {"value": n / sum(walls), "unit": "symbols/s", "cores": cores, "kind": "oracle",
            "value_1core": n / sum(cpus),
            "sample": f"{n} symbol(s) of {cfg.name} (per-step stages a1, a3-a6; ZF built untimed), fp64 numpy oracle "
                      f"over {cores} worker processes (1 BLAS thread each; FD-CNN per UE, precode/IDFT/GMP/receive "
                      f"per antenna block), wall {sum(walls):.1f} s; value_1core = symbols / summed task CPU time "
                      f"({sum(cpus):.1f} s)",
            "cpu_model": OP.cpu_model(), "affinity_cores": OP.host_cores()}


# ============================================================================ main arms
def init_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def batch_of(cfg, args):
    return args.batch or cfg.bench_batch or cfg.n_sym


def run_reference(args, cfg):
    """The reference arm: the fp64 oracle as it stands, on the host cores of rank 0 (the other
    ranks exit without work).  Each step = one OFDM symbol of the same workload (a bounded sample:
    a C5 symbol is ~45 s of single-core work), spread over all host cores."""
    from oracle import parallel as OP
    ws, rank, _ = init_dist()
    if rank != 0:
        return
    k = max(1, args.ref_step_symbols or (1 if cfg.name[:2] in ("C4", "C5") else 4))
    total_steps = args.warmup + args.steps
    inp = gen.make_inputs(cfg, list(range(total_steps * k)))
    times, cpus = [], []
    with OP.OracleRunner(cfg, inp) as r:
        for st in range(total_steps):
            w = c = 0.0
            for i in range(st * k, st * k + k):
                _, dw, dc = r.symbol(i)
                w += dw
                c += dc
            if st >= args.warmup:
                times.append(w)
                cpus.append(c)
        cores = r.workers
    total = sum(times)
    value = args.steps * k / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "symbols/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, ws, batch_of(cfg, args)),
        "cpu_baseline": {"value": value, "unit": "symbols/s", "cores": cores, "kind": "oracle",
                         "value_1core": args.steps * k / sum(cpus), "cpu_model": OP.cpu_model(),
                         "sample": f"{k} symbol(s) of {cfg.name} per step over {cores} worker processes (fp64 numpy "
                                   f"oracle as it stands, 1 BLAS thread each); value_1core from summed task CPU time"},
        "e2e": {"value": value, "unit": "symbols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, ws, batch):
    return {"workload": cfg.name, "U": cfg.U, "B": cfg.B, "N_ifft": cfg.N_ifft, "N_d": cfg.N_d, "M_qam": cfg.M_qam,
            "gmp": {"orders": list(cfg.orders), "L": cfg.L, "M": cfg.M}, "cnn_chans": list(cfg.chans),
            "seed": cfg.seed, "git_sha": git_sha(),
            "symbols_per_gpu_per_step": batch, "global_batch_symbols": batch * ws,
            "parallelism": f"symbol-batch x{ws}", "l2": "flushed between steps (256 MiB write outside the events)"}


def cnn_tc_issued_per_symbol(cfg):
    """FLOPs the tensor cores execute per OFDM symbol on the tensor-core FD-CNN path (conv_tc.cu),
    counted from the real MMA shapes: per 128-pixel tile of the zero-haloed image (n_tiles per UE
    image) and tap, the first layer (kind::tf32, K = 8: C_in = 2 padded) and the hidden layers
    (kind::f16, K = 16 steps over C_in) each issue A_hi.[W_hi | W_lo] (N = 2 C_out) and A_lo.W_hi
    (N = C_out); the last layer (C_out = 2) runs on the FP32 pipe.  Returns (tf32_flops, f16_flops)."""
    if cfg.head == "paper" or cfg.chans[1] < 16:
        return 0, 0
    S = cfg.S
    Wp = S + 2
    tiles = -(-(S * Wp) // 128)
    per_img_tf32 = per_img_f16 = 0
    for li, (ci, co) in enumerate(zip(cfg.chans[:-1], cfg.chans[1:])):
        if li == len(cfg.chans) - 2:
            break
        n = 3 * co                                       # N = 2 C_out + C_out
        if li == 0:
            per_img_tf32 += tiles * 9 * 2 * 128 * 8 * n
        else:
            per_img_f16 += tiles * 9 * 2 * 128 * ci * n
    return per_img_tf32 * cfg.U, per_img_f16 * cfg.U


def cnn_flop_per_symbol(cfg):
    """Algorithmic FD-CNN FLOPs per OFDM symbol: 2 x 9 C_in C_out per pixel and layer, S^2 pixels
    per UE image (P:180-195 counting convention, BASELINE network)."""
    if cfg.head == "paper":
        return 0
    return cfg.U * cfg.S ** 2 * sum(2 * 9 * a * b for a, b in zip(cfg.chans[:-1], cfg.chans[1:]))


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2205_05158_b200 import fdpd
    from paper_2205_05158_b200 import dist as D
    from paper_2205_05158_b200.chain import Chain, Shapes

    ws, rank, local = init_dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    fdpd.lib()
    fdpd.set_combine_path({"auto": 0, "simt": 1, "tc": 2}[args.combine])
    fdpd.set_gmp_path({"auto": 0, "simt": 1, "tc": 2}[args.gmp])
    n = batch_of(cfg, args)
    symbols = D.symbol_range(n, rank)          # Mode S, weak scaling
    inp = gen.make_inputs(cfg, symbols)

    impair = None
    if args.impair:
        impair = dict(clip=cfg.clip, pa_noise_std=cfg.pa_noise_std, awgn_n0=cfg.awgn_n0, csi_eta=cfg.csi_eta,
                      noise_key=inp["noise_key"], h_err=inp["h_err"])
    t_zf0 = time.perf_counter()
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], device=dev, max_batch=n,
               impair=impair, precode_math=args.precode_math)
    torch.cuda.synchronize()
    t_zf = time.perf_counter() - t_zf0
    if args.split_precode:
        ch.split_precode = True
    native = fdpd.NativeChain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=n,
                              device=dev)

    s = torch.from_numpy(inp["s"]).to(dev)
    idx = torch.from_numpy(inp["idx"]).to(dev)
    taps_all = torch.from_numpy(gen.channel_taps_per_symbol(cfg, symbols)).to(dev) if args.redraw else None
    counts = torch.zeros(3, dtype=torch.int64, device=dev)          # one step's counters
    total = torch.zeros(3, dtype=torch.int64, device=dev)           # summed over the timed steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sym0 = symbols[0]
    split = ch.split_precode and not (args.redraw or args.unfused)

    def step(ev=None):
        """ev: 4 events recorded after the CNN, the precode, the chain kernel and the combine."""
        counts.zero_()
        st = ch.dpd(s)
        if ev is not None:
            ev[0].record(stream)
        if split:
            X = ch.precode(st)
        if ev is not None:
            ev[1].record(stream)
        if args.redraw:
            XPA = ch.redraw_txrx(st, taps_all, sym0)       # batched per-symbol ZF + chain_txrx_ps
        elif args.unfused:
            y = ch.tx(st)
        elif split:
            _, XPA = ch.txrx_pre(X, sym0)
        else:
            _, XPA = ch.txrx(st, sym0)
        if ev is not None:
            ev[2].record(stream)
        if args.redraw:
            ch.redraw_combine(XPA, idx, counts=counts, sym0=sym0)
        elif args.unfused:
            ch.rx(y, idx, counts=counts)
        else:
            ch.combine(XPA, idx, counts=counts, sym0=sym0)
        if ev is not None:
            ev[3].record(stream)
        if ws > 1:
            D.allreduce_counts(counts)
        total.add_(counts)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    torch.cuda.synchronize()
    total.zero_()
    if ws > 1:
        dist.barrier()

    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [tuple(E() for _ in range(6)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step(ev=evs[i][1:5])
            evs[i][5].record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        total_h = total.cpu()
        if int(total_h[1]) != args.steps * ws * n * cfg.U * cfg.N_d:
            raise RuntimeError(f"step counters wrong: {total_h.tolist()}")
        # end-to-end through the C runtime (fd_chain_run_host*): pinned host inputs copied in, the
        # step, the SER counters copied back, every step
        s_h = torch.from_numpy(inp["s"]).pin_memory()
        i_h = torch.from_numpy(inp["idx"]).pin_memory()
        c_h = torch.zeros(3, dtype=torch.int64).pin_memory()
        e2e_ev = [(E(), E()) for _ in range(args.steps)]
        # the C runtime covers the default chain; impairments / per-symbol channels run the same
        # per-call path as the timed step, with the host copies added around it
        use_native = not (args.impair or args.redraw or args.unfused)
        s_d, i_d = torch.empty_like(s), torch.empty_like(idx)
        c_d = torch.zeros(3, dtype=torch.int64, device=dev)

        def reduce_host(ch_host):
            """all-reduce host counters through a persistent device buffer (Mode S counter sum)."""
            if ws > 1:
                c_d.copy_(ch_host, non_blocking=True)
                D.allreduce_counts(c_d)
                ch_host.copy_(c_d, non_blocking=True)

        for i in range(args.steps):
            flush.zero_()
            e2e_ev[i][0].record(stream)
            if use_native:
                native.run_host(s_h, i_h, c_h)
                reduce_host(c_h)
            else:
                s_d.copy_(s_h, non_blocking=True)
                i_d.copy_(i_h, non_blocking=True)
                counts.zero_()
                if args.redraw:
                    ch.step_redraw(s_d, i_d, taps_all, counts=counts, sym0=sym0)
                else:
                    ch.step(s_d, i_d, counts=counts, sym0=sym0, fused=not args.unfused)
                D.allreduce_counts(counts)
                c_h.copy_(counts, non_blocking=True)
            e2e_ev[i][1].record(stream)
        torch.cuda.synchronize()
        if int(c_h[1]) != ws * n * cfg.U * cfg.N_d:
            raise RuntimeError(f"e2e counters wrong: {c_h.tolist()}")
        # end-to-end from the QAM index stream (fd_chain_run_host_qam): only the uint16 indices
        # are copied in and the symbol mapping runs on the device
        e2e_q_ev = [(E(), E()) for _ in range(args.steps)] if use_native else []
        cq_h = torch.zeros(3, dtype=torch.int64).pin_memory()
        for i in range(len(e2e_q_ev)):
            flush.zero_()
            e2e_q_ev[i][0].record(stream)
            native.run_host_qam(i_h, cq_h)
            reduce_host(cq_h)
            e2e_q_ev[i][1].record(stream)
        torch.cuda.synchronize()
        if use_native and not torch.equal(cq_h, c_h):
            raise RuntimeError(f"e2e (QAM indices) counters {cq_h.tolist()} != {c_h.tolist()}")
    ms = sum(e[0].elapsed_time(e[5]) for e in evs)
    ms_e2e = sum(a.elapsed_time(b) for a, b in e2e_ev)
    ms_e2e_q = sum(a.elapsed_time(b) for a, b in e2e_q_ev) if e2e_q_ev else 0.0
    st_dpd = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    st_pre = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    st_tx = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    st_rx = statistics.mean(e[3].elapsed_time(e[4]) for e in evs)
    t = torch.tensor([ms, ms_e2e, st_tx, ms_e2e_q, st_dpd], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e, st_tx, ms_e2e_q, st_dpd = t.tolist()
    if rank != 0:
        dist.destroy_process_group()
        return

    total_symbols = n * ws * args.steps
    value = total_symbols / (ms / 1e3)
    pk = peaks()
    fp32_peak = 148 * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12       # TFLOP/s
    N = cfg.N_ifft
    fft_flop = 5 * N * int(np.log2(N)) * cfg.B
    if args.unfused:
        kern, tx_flop = "chain_tx (precode+IDFT+GMP)", chain_tx_flop_per_symbol(cfg)
    elif split:
        kern = "chain_txrx_pre (IDFT+GMP+receive DFT)"
        tx_flop = fft_flop + gmp_flop_per_sample(cfg) * N * cfg.B + fft_flop
    else:
        kern = "chain_txrx (precode+IDFT+GMP+receive DFT)"
        tx_flop = chain_tx_flop_per_symbol(cfg) + fft_flop
    achieved = tx_flop * n / (st_tx / 1e3) / 1e12
    bytes_sym = chain_bytes_per_symbol(cfg, fused=not args.unfused)
    hbm_achieved = bytes_sym * n * args.steps / (ms / 1e3) / 1e9
    if cfg.head == "paper":
        cnn_launches = 2                                   # conv + FC GEMM
    elif fdpd.lib().fdcnn_workspace_bytes(fdpd._ints(cfg.chans), len(cfg.chans) - 1, n, cfg.U, cfg.N_d) == 0:
        cnn_launches = 1                                   # whole network in shared memory
    else:
        cnn_launches = 2 * (len(cfg.chans) - 1)            # weight split + conv per layer
    chain_launches = 2 if split else 1                     # (+ precode)
    launches_per_step = cnn_launches + chain_launches + (2 if args.unfused else 1) + (3 if args.redraw else 0)
    # the tensor-core FD-CNN: 3 TF32 products per FP32-accurate MAC (hi/lo split), against the TF32
    # peak = measured bf16 x the guide's nominal TF32/BF16 ratio (1.1 / 2.25)
    cnn_flop = cnn_flop_per_symbol(cfg) * n
    cnn_tf32, cnn_f16 = cnn_tc_issued_per_symbol(cfg)
    cnn_equiv = (cnn_tf32 * 2.25 / 1.1 + cnn_f16) * n
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = oracle_sample(cfg, first_symbol=0)
    line = {
        "metric": METRIC, "value": value, "unit": "symbols/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator, workload/gen.py)",
        "config": dict(config_dict(cfg, ws, n), impairments=bool(args.impair),
                       channel=("per-symbol redraw, ZF in the step" if args.redraw else
                                "one realisation per run, ZF before timing"),
                       precode=("tensor cores, " + ch.precode_math if split and ch.precode_math != "simt"
                                else ("FP32 SIMT kernel" if split else "fused into the chain kernel")),
                       channel_sum={"auto": "FP32 SIMT (auto)", "simt": "FP32 SIMT", "tc": "tensor cores"}[args.combine]),
        "roofline": {"kernel": kern, "bound": "alu", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                     "traffic": measured_traffic(cfg, n, args),
                     "peak_src": f"derived: 148 SM x 128 FP32 lanes x 2 x {pk['sm_max_mhz']:.0f} MHz",
                     "flop_per_symbol": tx_flop, "ms_per_launch": st_tx},
        "roofline_cnn": ({"kernel": "fdcnn_forward (tcgen05: kind::tf32 first layer, kind::f16 hidden layers, "
                                    "hi/lo split operands; last layer FP32)", "bound": "tensor",
                          "algorithmic_tflops": cnn_flop / (st_dpd / 1e3) / 1e12,
                          # issued MMA work in f16-rate units (a TF32 FLOP costs 2.25/1.1 f16 FLOPs)
                          "achieved": cnn_equiv / (st_dpd / 1e3) / 1e12, "peak": pk["bf16_tflops"],
                          "unit": "TFLOP/s (f16 rate)", "frac": cnn_equiv / (st_dpd / 1e3) / 1e12 / pk["bf16_tflops"],
                          "issued_tf32_tflop_per_step": cnn_tf32 * n / 1e12, "issued_f16_tflop_per_step": cnn_f16 * n / 1e12,
                          "peak_src": "measured bf16 (MEASURED_PEAKS.json; f16 runs at the bf16 rate; TF32 at the "
                                      "guide's nominal 1.1/2.25 of it)",
                          "ms_per_step": st_dpd}
                         if cnn_flop and cfg.chans[1] >= 32 else None),
        "hbm": {"algorithmic_bytes_per_symbol": bytes_sym, "achieved_GBps": hbm_achieved, "peak_GBps": pk["hbm_gbs"],
                "frac": hbm_achieved / pk["hbm_gbs"], "peak_src": pk["src"]},
        "stage_ms": {"fdcnn": st_dpd, "precode": st_pre if split else 0.0,
                     ("chain_tx" if args.unfused else ("chain_txrx_pre" if split else "chain_txrx")): st_tx,
                     ("ue_receive_ser" if args.unfused else "ue_combine_ser"): st_rx, "zf_build_once_s": t_zf},
        "counters": {"errors": int(total_h[0]), "total": int(total_h[1]), "near_boundary": int(total_h[2])},
        "cpu_baseline": cpu,
        "e2e": ({"value": total_symbols / (ms_e2e_q / 1e3), "unit": "symbols/s",
                 "h2d_bytes_per_step": int(inp["idx"].nbytes), "d2h_bytes_per_step": 24,
                 "api": "fd_chain_run_host_qam (host QAM indices in, SER counters out; symbol mapping on "
                        "the device)"} if ms_e2e_q > 0 else
                {"value": total_symbols / (ms_e2e / 1e3), "unit": "symbols/s",
                 "h2d_bytes_per_step": int(inp["s"].nbytes + inp["idx"].nbytes), "d2h_bytes_per_step": 24,
                 "api": "per-call path with host copies"}),
        "e2e_symbols_in": {"value": total_symbols / (ms_e2e / 1e3), "unit": "symbols/s",
                           "h2d_bytes_per_step": int(inp["s"].nbytes + inp["idx"].nbytes), "d2h_bytes_per_step": 24,
                           "api": "fd_chain_run_host (host complex64 symbols + indices in)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_antenna(args, cfg):
    """Mode A (BASELINE configs[4]): antenna rows [b0, b0 + B/N) per rank, FD-CNN on
    the rank's n symbols, all_gather_into_tensor of s_tilde, precode -> IDFT/GMP/receive DFT on the
    local antennas for the world batch of N n symbols, partial channel sum, reduce_scatter_tensor
    (each rank gets y_hat of its own symbols), slicing, counter all-reduce; two micro-batches so the
    collectives overlap the next micro-batch's compute.  Weak scaling: per GPU, n symbols of CNN and
    N n symbols x B/N antennas of chain = the 1-GPU step's work."""
    import torch
    import torch.distributed as dist

    from paper_2205_05158_b200 import fdpd
    from paper_2205_05158_b200 import dist as D
    from paper_2205_05158_b200.chain import AntennaOps, Chain, Shapes

    ws, rank, local = init_dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    fdpd.lib()
    fdpd.set_combine_path({"auto": 0, "simt": 1, "tc": 2}[args.combine])
    fdpd.set_gmp_path({"auto": 0, "simt": 1, "tc": 2}[args.gmp])
    n = batch_of(cfg, args)
    micro = 2 if n % 2 == 0 else 1
    symbols = D.symbol_range(n, rank)
    inp = gen.make_inputs(cfg, symbols)
    b0, B_loc = D.antenna_shard(cfg.B, ws, rank)
    math = args.precode_math
    t0 = time.perf_counter()
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], device=dev,
               max_batch=ws * n // micro, b0=b0, B_loc=B_loc, precode_math=math)
    torch.cuda.synchronize()
    t_zf = time.perf_counter() - t0
    chain_ev = []
    ops = AntennaOps(ch, events=chain_ev)
    # Exchange of the partial received signals: fused into the channel-sum kernel over peer memory
    # (ue_combine_peer; auto: where it applies and the peer mappings validate), else NCCL
    # reduce_scatter_tensor.
    peer, exchange = None, "NCCL reduce_scatter_tensor"
    if args.exchange != "nccl" and ops.peer_ok():
        try:
            peer = D.PeerExchange(micro, n // micro, cfg.U, cfg.N_d, dev)
            exchange = "fused into ue_combine_peer (peer memory, CUDA IPC mappings)"
        except Exception as e:                      # every rank fails or none: the validation is collective
            if args.exchange == "peer":
                raise
            print(f"[bench] peer exchange unavailable ({e}); using NCCL", file=sys.stderr)
    step = D.AntennaShardedStep(ops, n, cfg.U, cfg.N_d, micro=micro, peer=peer,
                                alloc=lambda shp: torch.empty(shp, dtype=torch.complex64, device=dev))
    s = torch.from_numpy(inp["s"]).to(dev)
    idx = torch.from_numpy(inp["idx"]).to(dev)
    counts = torch.zeros(3, dtype=torch.int64, device=dev)
    total = torch.zeros(3, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        counts.zero_()
        step.step(s, idx, counts)
        flush.zero_()
    torch.cuda.synchronize()
    chain_ev.clear()
    if ws > 1:
        dist.barrier()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [(E(), E()) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            counts.zero_()
            step.step(s, idx, counts)
            total.add_(counts)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        n_chain = len(chain_ev)
        ms_chain = sum(a.elapsed_time(b) for a, b in chain_ev) / max(1, n_chain)
        chain_ev.clear()
        ops.events = None
        if ws > 1:
            dist.barrier()
        total_h = total.cpu()
        if int(total_h[1]) != args.steps * ws * n * cfg.U * cfg.N_d:
            raise RuntimeError(f"step counters wrong: {total_h.tolist()}")
        # end to end: this rank's QAM symbols and indices from pinned host memory, the step, the
        # world SER counters back to the host, every step
        s_h = torch.from_numpy(inp["s"]).pin_memory()
        i_h = torch.from_numpy(inp["idx"]).pin_memory()
        c_h = torch.zeros(3, dtype=torch.int64).pin_memory()
        s_d, i_d = torch.empty_like(s), torch.empty_like(idx)
        e2e = [(E(), E()) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            e2e[i][0].record(stream)
            s_d.copy_(s_h, non_blocking=True)
            i_d.copy_(i_h, non_blocking=True)
            counts.zero_()
            step.step(s_d, i_d, counts)
            c_h.copy_(counts, non_blocking=True)
            e2e[i][1].record(stream)
        torch.cuda.synchronize()
        if int(c_h[1]) != ws * n * cfg.U * cfg.N_d:
            raise RuntimeError(f"e2e counters wrong: {c_h.tolist()}")
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_e2e = sum(a.elapsed_time(b) for a, b in e2e)
    t = torch.tensor([ms, ms_e2e, ms_chain], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e, ms_chain = t.tolist()
    if rank != 0:
        dist.destroy_process_group()
        return
    total_symbols = n * ws * args.steps
    pk = peaks()
    fp32_peak = 148 * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    N = cfg.N_ifft
    flop_sym_ant = 2 * 5 * N * int(np.log2(N)) + gmp_flop_per_sample(cfg) * N     # IDFT + GMP + receive DFT
    achieved = flop_sym_ant * (ws * n // micro) * B_loc / (ms_chain / 1e3) / 1e12
    comm = 8 * ws * n * cfg.U * cfg.N_d
    line = {
        "metric": METRIC, "value": total_symbols / (ms / 1e3), "unit": "symbols/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator, workload/gen.py)",
        "config": dict(config_dict(cfg, ws, n), parallelism=f"antenna x{ws} (Mode A: {B_loc} antennas per GPU)",
                       precode=("tensor cores, " + math) if math != "simt" else "FP32 SIMT kernel",
                       micro_batches=micro, world_batch_symbols=ws * n,
                       collectives="all_gather_into_tensor(s_tilde) per micro-batch (NCCL, async, overlapped) + "
                                   "int64 counter all_reduce; y_hat partials: " + exchange,
                       comm_bytes_per_rank_per_step={"all_gather_in": comm * (ws - 1) // ws,
                                                     "reduce_scatter_out": comm * (ws - 1) // ws}),
        "roofline": {"kernel": "chain_txrx_pre (IDFT+GMP+receive DFT)", "bound": "alu", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": None,
                     "peak_src": f"derived: 148 SM x 128 FP32 lanes x 2 x {pk['sm_max_mhz']:.0f} MHz",
                     "ms_per_launch": ms_chain},
        "counters": {"errors": int(total_h[0]), "total": int(total_h[1]), "near_boundary": int(total_h[2])},
        "stage_ms": {"zf_build_once_s": t_zf},
        "cpu_baseline": None,
        "e2e": {"value": total_symbols / (ms_e2e / 1e3), "unit": "symbols/s",
                "h2d_bytes_per_step": int(inp["s"].nbytes + inp["idx"].nbytes), "d2h_bytes_per_step": 24,
                "api": "Mode A step (per-call path) with host copies of each rank's symbols and indices"},
        "gpu_launches": None,
        "clocks": clk.summary(),
    }
    cnn_l = 2 * (len(cfg.chans) - 1)
    line["gpu_launches"] = args.steps * micro * (cnn_l + (2 if math != "simt" else 2) + 2)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--batch", type=int, default=0, help="symbols per GPU per step (default: the config's bench batch)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-step-symbols", type=int, default=0,
                    help="oracle symbols per --impl reference step (default 1 at C4/C5, else 4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="chain_tx + ue_receive_ser instead of chain_txrx")
    ap.add_argument("--impair", action="store_true", help="PA clip + noise, AWGN, imperfect CSI (NEXT f3)")
    ap.add_argument("--redraw", action="store_true", help="per-symbol channel redraw, ZF on the hot path (NEXT f4)")
    ap.add_argument("--split-precode", action="store_true", help="precode kernel + chain_txrx_pre")
    ap.add_argument("--precode-math", default="auto", choices=["auto", "simt", "tf32", "fp32tc"],
                    help="split-path precode: FP32 SIMT, TF32 tensor cores, or FP32-accurate split-TF32 tensor cores")
    ap.add_argument("--combine", default="auto", choices=["auto", "simt", "tc"],
                    help="channel sum: auto (= the FP32 SIMT kernels), simt, or tc (tensor cores for 9 <= U <= 32)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                    help="Mode A: partial received signals through peer memory from the channel-sum kernel, or NCCL")
    ap.add_argument("--gmp", default="auto", choices=["auto", "simt", "tc"],
                    help="GMP of the N = 16384 cluster chain: auto, FP32 SIMT, or tensor cores (C4 / C5 shape)")
    ap.add_argument("--mode", default="auto", choices=["auto", "symbol", "antenna"],
                    help="multi-GPU partitioning: symbol batches (Mode S) or antennas (Mode A); auto = antenna "
                         "for C5 at N > 1 (BASELINE configs[4]), else symbol")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    cfg = configs.get(args.config)
    if args.impair:
        cfg = configs.impaired(cfg)
    if (args.impair or args.redraw) and args.unfused:
        ap.error("--impair/--redraw run on the fused path only")
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    antenna = args.mode == "antenna" or (args.mode == "auto" and ws > 1 and cfg.name == "C5")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif antenna:
        if args.impair or args.redraw or args.unfused:
            ap.error("Mode A runs the default chain only")
        run_antenna(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
