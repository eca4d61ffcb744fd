"""bench.py -- throughput of the batch-invariant log-prob + TIS/RS hot path on B200.

    python bench.py [--gpus N --steps K --warmup W --config c2 --scaling strong --impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one pass of the whole hot path over one batch:
tim_logprob (lm_head GEMM + fused online log-softmax / gather / entropy + slice merge) on the
rank's tokens, then tim_correct (delta, TIS, sequence-RS K3 with the paper's tau values,
statistics; NCCL all-gather of exact partials when N > 1).  Default workload: C2 (Qwen3-8B head,
d = 4096, 256 x 8192 tokens), the largest single-GPU config of BASELINE.json; C1 and C3 are
reported as extra keys at N = 1.  Strong scaling (default): the config's global batch is cut
into N token shards (cuts inside sequences); value = global tokens / max-rank time.

Metric (BASELINE.json): logprob tokens/sec at V = 151936; also max |dlogp| across batch shapes.
Inputs are synthetic (synth/), resident in HBM for `value`; `e2e` re-times the step through the
public API from pinned host buffers (H2D of the inputs and D2H of the results inside the timing).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

# The reference arm (--impl reference) runs the CPU oracle on rank 0 alone: give its BLAS every
# host core even when the launcher (torchrun) pinned OMP_NUM_THREADS=1 for the per-GPU ranks.
# This has to happen before numpy / torch load OpenBLAS.
if "--impl" in sys.argv and "reference" in sys.argv and os.environ.get("RANK", "0") == "0":
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[_v] = str(os.cpu_count() or 1)
import statistics
import subprocess
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
KERNELS_PER_STEP = 5  # logprob fwd + merge, correct local + finish + zero
_SMS = 148            # B200 SMs (the clock-peak figure below; the kernels query the device themselves)


def _peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _ncu_tensor_pct(config: str):
    """ncu tensor-pipe activity of the logprob kernel on this config, from the committed --set full
    summary (None when no capture of this config is committed)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_logprob_summary.json")) as f:
            d = json.load(f)
        v = d.get(f"tensor_pipe_pct_{config}")
        if v is None and config == "c1":
            v = d["metrics"]["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]
        return None if v is None else float(v)
    except Exception:
        return None


def _kernel_clock_mhz(tim, dev):
    """Average SM clock of the last tim_logprob launch on this stream, measured inside the kernel
    (CTA 0: clock64 and globaltimer at its start and end, workspace header reserved[1..4]) -- the
    clock the power cap actually sustained, which nvidia-smi's 200-ms samples can overstate."""
    try:
        key = (str(dev), torch.cuda.current_stream(dev).cuda_stream, "logprob")
        ws = tim._ws_cache.get(key)
        if ws is None:
            return None
        h = ws[:64].view(torch.int64).cpu().tolist()  # WsHeader: bad_inv, counter|pad, reserved[0..5]
        cyc, ns = h[5] - h[3], h[6] - h[4]            # clk = reserved[1..4]: {cyc0, ns0, cyc1, ns1}
        return round(cyc / ns * 1e3, 1) if ns > 0 and cyc > 0 else None
    except Exception:
        return None


def _traffic(config: str):
    """dram bytes per launch of the logprob kernel on this config, from the committed ncu --set
    full summary (None when no capture of this config is committed)."""
    p = os.path.join(ROOT, "profiles", "ncu_logprob_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"dram_bytes_per_launch_{config}")
    except Exception:
        return None


def _hbm_traffic(key: str, n: int):
    """dram bytes per pass-1 launch of the correction / PPO kernel at 2^27 tokens, from the
    committed ncu --set full summary (None for another size or when absent)."""
    if n != 1 << 27:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_hbm_kernels_summary.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def build_workload(cfg, scaling, world, rank, device):
    """The rank's slice of the workload.

    strong: the config's global batch (n_seq x seq_len tokens) is cut into P token shards
            (tim.shard_range: floor(r N / P) rounded to 256 rows, cuts inside sequences -- the
            sequences straddle ranks); rows are drawn chunk-wise (synth.global_rows)
            so every partition sees the same global batch.  P = 1 is the whole config.
    weak:   every rank scores its own config-sized batch (sequences rank*S .. (rank+1)*S - 1).
    Returns (W, H, ids, tok_begin, cu_global, resp_mask_local, n_global)."""
    from paper_2605_14220_b200 import tim

    W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device=device)  # replicated lm_head
    if scaling == "strong":
        n_glob = cfg.n_tok
        a, b = tim.shard_range(n_glob, world, rank)
        H, ids = synth.global_rows(n_glob, cfg.hidden, cfg.vocab, cfg.seed, a, b, W, device=device)
        cu = synth.cu_seqlens(cfg.n_seq, cfg.seq_len)
        mask = synth.resp_mask(cu, cfg.prompt_len)[a:b]
        return W, H, ids, a, cu.to(device), mask.to(device), n_glob
    seed = cfg.seed + 1000 * rank
    ids = synth.token_ids(cfg.n_tok, cfg.vocab, seed, device=device)
    H = synth.hidden_states(cfg.n_tok, cfg.hidden, seed, device=device, weight=W, ids=ids, mode="peaked")
    cu = synth.cu_seqlens(cfg.n_seq * world, cfg.seq_len)
    mask = synth.resp_mask(synth.cu_seqlens(cfg.n_seq, cfg.seq_len), cfg.prompt_len)
    return W, H, ids, rank * cfg.n_tok, cu.to(device), mask.to(device), world * cfg.n_tok


def run_ours(args):
    from paper_2605_14220_b200 import tim

    world, rank, local = _dist()
    if args.tuning:
        vals = [int(x) for x in args.tuning.split(",")]
        tim.debug_set_tuning(*vals[:4])
        if len(vals) > 4:
            tim.debug_set_schedule(vals[4], vals[5] if len(vals) > 5 else 0)
    if args.max_pairs:
        tim.debug_set_kernel(True, args.max_pairs)
    if args.cluster_pairs:
        tim.debug_set_cluster(args.cluster_pairs)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    comm = tim.Comm() if world > 1 else None
    # application-level L2 setup: a persisting set-aside for the evict_last H tiles of the log-prob
    # kernel (include/tim.h tim_l2_persisting; profiles/r02_c2_bimodal.txt)
    l2_granted = tim.l2_persisting(args.l2_persist_mb << 20, dev) if args.l2_persist_mb >= 0 else None
    # the HBM-bound kernels are timed alone, first (before the long tensor-bound steps heat the
    # GPU into its power-capped state), against the burst copy bandwidth
    hbm_lines = {}
    if args.correction_tokens > 0:
        peaks0, peak_src0 = _peaks()
        hbm_lines["correction_roofline"] = correction_roofline(tim, dev, args.correction_tokens, peaks0, peak_src0)
        hbm_lines["ppo_roofline"] = ppo_roofline(tim, dev, args.correction_tokens, peaks0, peak_src0)
        torch.cuda.empty_cache()
    cfg = synth.CONFIGS[args.config]
    if args.n_seq:
        import dataclasses
        cfg = dataclasses.replace(cfg, n_seq=args.n_seq)
    out = measure(tim, cfg, args, world, rank, local, dev, comm, args.steps, args.warmup, full=True)
    out.update(hbm_lines)
    if l2_granted is not None:
        out["config"]["l2_persisting_mb"] = round(l2_granted / 2**20, 1)
    # the other single-GPU configs of BASELINE.json as extra keys (N = 1): each its own step
    # timing and roofline; the headline stays the config named in config.workload
    if world == 1 and args.extra_configs:
        extra = {}
        for name, steps in (("c1", 5), ("c3", 2)):
            if name == cfg.name:
                continue
            torch.cuda.empty_cache()
            e = measure(tim, synth.CONFIGS[name], args, world, rank, local, dev, comm, steps, 3, full=False)
            extra[name] = {k: e[k] for k in ("value", "unit", "ms_per_step", "steps", "warmup", "config", "roofline",
                                             "clocks", "max_abs_dlogp_across_shapes", "correction_stats",
                                             "scaling")}
        out["extra_configs"] = extra
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def measure(tim, cfg, args, world, rank, local, dev, comm, steps, warmup, full):
    scaling = args.scaling
    W, H, ids, tok_begin, cu, mask, n_glob = build_workload(cfg, scaling, world, rank, dev)
    N = H.shape[0]
    ccfg = tim.PRESETS["tis-srs-k3-corr-ratio"]

    # rollout-side log-probs: the same head with a P3 perturbation (setup, untimed)
    lp0, _ = tim.logprob(H, W, ids)
    lp_roll = synth.perturb_laplace_mix(lp0, cfg.seed + rank)
    del lp0
    lp = torch.empty(N, dtype=torch.float32, device=dev)
    ent = torch.empty(N, dtype=torch.float32, device=dev)
    S_glob = cu.numel() - 1
    cout = {"tis_w": torch.empty(N, dtype=torch.float32, device=dev),
            "tok_keep": torch.empty(N, dtype=torch.uint8, device=dev),
            "seq_keep": torch.empty(S_glob, dtype=torch.uint8, device=dev),
            "coeff": torch.empty(N, dtype=torch.float32, device=dev),
            "seq_score": torch.empty(S_glob, dtype=torch.float64, device=dev),
            "stats_raw": torch.zeros(tim.STATS_BYTES, dtype=torch.uint8, device=dev)}
    status = tim.new_status(dev)
    # the logprob kernels run on the caller's current stream: time them with events on that stream
    cur = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(cur)
        tim.logprob(H, W, ids, out=(lp, ent), status=status)
        if ev is not None:
            ev[1].record(cur)
        tim.correct(lp, lp_roll, cu, ccfg, mask, tok_begin=tok_begin, comm=comm, status=status,
                    return_stats=False, out=cout)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0.record(cur)
    for k in range(steps):
        step(evs[k])
    t1.record(cur)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    clk["sm_mhz_in_kernel"] = _kernel_clock_mhz(tim, dev)
    try:  # the SM -> die map behind the die-aware M-tile groups (state 1 = probed and valid)
        st_dm, die = tim.debug_die_map()
        clk["die_map"] = {"state": st_dm, "die1_sms": int(sum(die))}
    except Exception:
        pass
    ms = t0.elapsed_time(t1)
    lp_ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    if world > 1:
        t = torch.tensor([ms, lp_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, lp_ms = t.tolist()
    code, first = tim.read_status(status)
    assert code == 0, f"device status {code} at {first}"
    stats = tim.stats_from_bytes(cout["stats_raw"])

    # invariance (untimed): a sample of rows re-scored alone and in another pack size, bitwise
    samp = torch.arange(0, N, max(1, N // 64), device=dev)[:64]
    ref_bits = lp[samp].view(torch.int32)
    max_shape_diff = 0.0
    for r in samp[:16].tolist():
        a, _ = tim.logprob(H[r:r + 1], W, ids[r:r + 1])
        max_shape_diff = max(max_shape_diff, abs(a.item() - lp[r].item()))
    a, _ = tim.logprob(H[samp], W, ids[samp])
    if not torch.equal(a.view(torch.int32), ref_bits):
        max_shape_diff = max(max_shape_diff, (a - lp[samp]).abs().max().item())

    peaks, peak_src = _peaks()
    flop = 2.0 * cfg.vocab * cfg.hidden * N
    achieved = flop / (lp_ms / 1e3) / 1e12
    peak = float(peaks["bf16_tflops_sustained"])
    value = (n_glob if scaling == "strong" else world * N) * steps / (ms / 1e3)
    if scaling == "strong":
        par = f"dp{world} (global batch token-sharded, cuts inside sequences)"
        wl = (f"{cfg.name}: Qwen3-shaped lm_head d={cfg.hidden}, V={cfg.vocab}, global batch {cfg.n_seq} seqs x "
              f"{cfg.seq_len} tokens over {world} GPU(s); logprob + entropy + tis-srs-k3-corr-ratio correction")
    else:
        par = f"dp{world} (token-sharded, a config-sized batch per GPU)"
        wl = (f"{cfg.name}: Qwen3-shaped lm_head d={cfg.hidden}, V={cfg.vocab}, {cfg.n_seq} seqs x "
              f"{cfg.seq_len} tokens per GPU; logprob + entropy + tis-srs-k3-corr-ratio correction")
    out = {
        "metric": "logprob tokens/sec at V=151936 (1/2/4/8 B200); max |dlogp| across batch shapes",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": ms / steps,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "bf16 inputs, fp32 tensor-core accumulate (tcgen05 kind::f16); fp64 correction",
        "data": "synthetic (synth/: peaked-mode hidden states, N(0,0.02^2) head, seeded)",
        "config": {
            "workload": wl, "hidden": cfg.hidden, "vocab": cfg.vocab, "n_seq": cfg.n_seq, "seq_len": cfg.seq_len,
            "tokens_this_gpu": N, "global_batch_tokens": n_glob, "parallelism": par,
            "l2": "inputs larger than L2 (H %.2f GB/GPU, W %.2f GB): no flush needed" % (N * cfg.hidden * 2 / 1e9,
                                                                                      W.numel() * 2 / 1e9),
        },
        "max_abs_dlogp_across_shapes": max_shape_diff,
        "gpu_launches": KERNELS_PER_STEP * steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "frac_of_burst": achieved / float(peaks["bf16_tflops"]),
                     "peak_source": peak_src + " bf16_tflops_sustained", "traffic": _traffic(cfg.name),
                     "ncu_tensor_pipe_pct": _ncu_tensor_pct(cfg.name),
                     "kernel": "tim_logprob (tcgen05 GEMM + fused epilogue + slice merge)",
                     "kernel_ms": lp_ms, "algorithmic_flop_per_token": 2 * cfg.vocab * cfg.hidden,
                     "tokens_per_launch": N,
                     # the tensor pipe's peak at the clock the kernel actually ran at (in-kernel
                     # clock64 / globaltimer): 148 SMs x 8192 dense bf16 flop per SM-cycle (from ncu:
                     # flops / tensor-active cycles); frac_of_clock_peak = what the power cap leaves
                     "frac_of_clock_peak": (achieved / (_SMS * 8192 * clk["sm_mhz_in_kernel"] * 1e-6))
                     if clk.get("sm_mhz_in_kernel") else None},
        "clocks": clk,
        "correction_stats": {k: stats[k] for k in ("n_resp_tok", "n_truncated", "n_seq_rejected", "max_abs_delta",
                                                     "mean_abs_delta", "mean_k3")},
    }
    if not full:
        return out

    # small-batch latency (rollout-side scoring): one call on the first n rows, n <= one M-tile
    small = {}
    for n_small in (1, 64, 256):
        lps = torch.empty(n_small, device=dev)
        ens = torch.empty(n_small, device=dev)
        for _ in range(3):
            tim.logprob(H[:n_small], W, ids[:n_small], out=(lps, ens))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(10):
            tim.logprob(H[:n_small], W, ids[:n_small], out=(lps, ens))
        e1.record(cur)
        torch.cuda.synchronize()
        small[str(n_small)] = round(e0.elapsed_time(e1) / 10, 4)
        assert torch.equal(lps.view(torch.int32), lp[:n_small].view(torch.int32))  # batch invariance
    out["small_batch_latency_ms"] = {"n_tok": small, "note": "tim_logprob on the first n rows of the batch, "
                                     "bitwise equal to their logp in the full batch"}

    # NEXT-1 rollout-side twin on the same batch: draw throughput and the zero-mismatch check
    if args.sample_bench:
        keys = (torch.arange(N, device=dev, dtype=torch.int64) << 32) | rank
        for _ in range(2):
            sid, slp, sent = tim.sample(H, W, keys, seed=20260001)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(3):
            sid, slp, sent = tim.sample(H, W, keys, seed=20260001)
        e1.record(cur)
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1) / 3
        rlp, rent = tim.logprob(H, W, sid)
        same = bool(torch.equal(rlp.view(torch.int32), slp.view(torch.int32)) and
                    torch.equal(rent.view(torch.int32), sent.view(torch.int32)))
        out["sample_twin"] = {"tokens_per_s": N / (sms / 1e3), "ms": sms,
                              "tflops": 2.0 * cfg.vocab * cfg.hidden * N / (sms / 1e3) / 1e12,
                              "logp_bitwise_equal_to_logprob": same,
                              "kernel": "tim_sample (tcgen05 GEMM + online LSE + Philox Gumbel-max epilogue)"}
        del sid, slp, sent, rlp, rent, keys
        torch.cuda.empty_cache()

    # NEXT-3 head backward on one token block of the batch (dL/dlogp = 1, dL/dH = 0.01)
    if args.backward_bench:
        out["head_backward"] = backward_bench(tim, cfg, H, W, ids, dev, cur)
        torch.cuda.empty_cache()

    # end to end through the public API from pinned host buffers
    Hh = H.cpu().pin_memory()
    if args.e2e_steps > 0:
        idsh = ids.cpu().pin_memory()
        rollh = lp_roll.cpu().pin_memory()
        maskh = mask.cpu().pin_memory()
        cuh = cu.cpu().pin_memory()
        del H
        torch.cuda.empty_cache()

        def e2e_step():
            lph, enth = tim.logprob(Hh, W, idsh, device=dev)
            res = tim.correct(lph, rollh, cuh, ccfg, maskh, tok_begin=tok_begin, comm=comm, device=dev)
            return lph, enth, res

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(args.e2e_steps):
            lph, enth, res = e2e_step()
        e1.record(cur)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = t.item()
        h2d = Hh.numel() * 2 + idsh.numel() * 8 + 2 * N * 4 + maskh.numel() + cuh.numel() * 8
        d2h = 2 * N * 4 + N * 4 + N + S_glob + N * 4 + S_glob * 8 + tim.STATS_BYTES
        n_e2e = n_glob if scaling == "strong" else world * N
        out["e2e"] = {"value": n_e2e * args.e2e_steps / (ems / 1e3), "unit": "tokens/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                      "ms_per_step": ems / args.e2e_steps}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"], out["max_abs_dlogp_vs_oracle"] = cpu_baseline(cfg, W, Hh, ids, lp, lp_roll, mask,
                                                                            args.cpu_seconds)
    return out


def backward_bench(tim, cfg, H, W, ids, dev, cur):
    nb = min(H.shape[0], 14080)
    gl = torch.ones(nb, device=dev)
    ge = torch.full((nb,), 0.01, device=dev)
    for _ in range(2):
        dh, dw = tim.head_backward(H[:nb], W, ids[:nb], gl, ge)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(3):
        dh, dw = tim.head_backward(H[:nb], W, ids[:nb], gl, ge)
    e1.record(cur)
    torch.cuda.synchronize()
    bms = e0.elapsed_time(e1) / 3
    # the trainer-side variant: entropy / lse2 saved by the forward (tim_logprob_saved)
    _, sent, slse2 = tim.logprob_saved(H[:nb], W, ids[:nb])
    for _ in range(2):
        dh, dw = tim.head_backward(H[:nb], W, ids[:nb], gl, ge, saved=(sent, slse2))
    e0.record(cur)
    for _ in range(3):
        dh, dw = tim.head_backward(H[:nb], W, ids[:nb], gl, ge, saved=(sent, slse2))
    e1.record(cur)
    torch.cuda.synchronize()
    sbms = e0.elapsed_time(e1) / 3
    return {"tokens": nb, "ms": bms, "tokens_per_s": nb / (bms / 1e3),
            "tflops_effective": 4 * 2.0 * cfg.vocab * cfg.hidden * nb / (bms / 1e3) / 1e12,
            "note": "4 passes of 2 V d flop per token: forward, gradient epilogue (logits recomputed), "
                    "dH = G W and dW = G^T H (hand-written tcgen05 GEMMs, csrc/gemm.cu)",
            "kernel": "tim_head_backward",
            "saved": {"ms": sbms, "tokens_per_s": nb / (sbms / 1e3),
                      "tflops_effective": 3 * 2.0 * cfg.vocab * cfg.hidden * nb / (sbms / 1e3) / 1e12,
                      "kernel": "tim_head_backward_saved (forward's entropy / lse2 saved: 3 passes)"}}


def H_bytes(cfg):
    return cfg.n_tok * cfg.hidden * 2


def ppo_roofline(tim, dev, n, peaks, peak_src, reps=10):
    """Standalone tim_ppo_loss (NEXT-2) at n tokens weighted by correction coefficients: 25
    algorithmic bytes per token (read lp_cur, lp_old, advantage, coeff; write loss, grad, clip flag)."""
    S = n // 4096
    cu = synth.cu_seqlens(S, 4096).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(20260005)
    old = -torch.empty(n, device=dev).exponential_(0.7, generator=g)
    cur = synth.policy_move(old, 20260005, sd=0.05)
    adv = torch.randn(n, device=dev, generator=g)
    coeff = torch.where(torch.arange(n, device=dev) % 4096 >= 1024, 1.0, 0.0).float()
    cfg = tim.PPOConfig(eps=0.2)
    for _ in range(3):
        tim.ppo_loss(cur, old, adv, cu, cfg, coeff=coeff, return_stats=False)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        tim.ppo_loss(cur, old, adv, cu, cfg, coeff=coeff, return_stats=False)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]
    gbs = 25.0 * n / (ms / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    return {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "traffic": _hbm_traffic("ppo_local_dram_bytes_2e27", n), "n_tok": n, "ms": ms,
            "algorithmic_bytes_per_token": 25, "kernel": "tim_ppo_loss (ppo_local + finish, median of %d)" % reps}


def correction_roofline(tim, dev, n, peaks, peak_src, reps=10):
    """Standalone tim_correct (tis-srs-k3-corr-ratio, 4096-token sequences, 3/4 response) at n
    tokens: 18 algorithmic bytes per token (read 2 fp32 + u8 mask, write fp32 w + u8 keep + fp32
    coeff) vs the measured HBM copy bandwidth.  Inputs (1.2 GB at 2^27) exceed L2."""
    S = n // 4096
    cu = synth.cu_seqlens(S, 4096).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(20260004)
    den = -torch.empty(n, device=dev).exponential_(0.7, generator=g)
    num = synth.perturb_laplace_mix(den, 20260004)
    mask = (torch.arange(n, device=dev) % 4096 >= 1024).to(torch.uint8)
    cfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
    out = {"tis_w": torch.empty(n, dtype=torch.float32, device=dev),
           "tok_keep": torch.empty(n, dtype=torch.uint8, device=dev),
           "seq_keep": torch.empty(S, dtype=torch.uint8, device=dev),
           "coeff": torch.empty(n, dtype=torch.float32, device=dev),
           "seq_score": torch.empty(S, dtype=torch.float64, device=dev),
           "stats_raw": torch.zeros(tim.STATS_BYTES, dtype=torch.uint8, device=dev)}
    for _ in range(3):
        tim.correct(num, den, cu, cfg, mask, return_stats=False, out=out)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        tim.correct(num, den, cu, cfg, mask, return_stats=False, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]
    # algorithmic bytes: 18 per token for pass 1 (a5) + 4 per token of a rejected sequence for the
    # coefficient zeroing (a7: "4 B/token only for tokens of rejected sequences")
    keep = out["seq_keep"].to(torch.int64)
    lens = (cu[1:] - cu[:-1]).to(torch.int64)
    n_rej_tok = int(((1 - keep) * lens).sum().item())
    bpt = 18.0 + 4.0 * n_rej_tok / n
    gbs = bpt * n / (ms / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    return {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "traffic": _hbm_traffic("correct_local_dram_bytes_2e27", n),
            "n_tok": n, "ms": ms, "algorithmic_bytes_per_token": bpt, "tokens_in_rejected_sequences": n_rej_tok,
            "peak_source": peak_src + " hbm_gbs",
            "kernel": "tim_correct (correct_local + finish + zero, median of %d)" % reps}


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, W, Hh, ids, lp_gpu, lp_roll, mask, seconds):
    """The fp64 oracle as it stands, on the host cores, over a bounded sample of the workload."""
    import math

    import numpy as np

    from oracle import correct as oc
    from oracle.logprob import logprob_entropy

    N = cfg.n_tok
    Wc = W.cpu()
    rows = torch.randperm(N, generator=torch.Generator().manual_seed(3))[:4096]
    done, t_lp, dmax = 0, 0.0, 0.0
    while t_lp < seconds * 0.6 and done < rows.numel():
        r = rows[done:done + 32]
        h = Hh[r]
        idr = ids.cpu()[r]
        t = time.perf_counter()
        olp, _ = logprob_entropy(h, Wc, idr, row_chunk=32)
        t_lp += time.perf_counter() - t
        dmax = max(dmax, float(np.abs(lp_gpu.cpu()[r].double().numpy() - olp).max()))
        done += r.numel()
    # correction oracle on whole sequences of the same batch
    ocfg = oc.Cfg(tis=True, tis_cap=2.0, log_tis_cap=math.log(2.0), seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM,
                  tau_seq=1e-3)
    n_corr = min(N, cfg.seq_len * 8)
    cu = synth.cu_seqlens(n_corr // cfg.seq_len, cfg.seq_len).numpy()
    t = time.perf_counter()
    oc.correct(lp_gpu[:n_corr].cpu().numpy(), lp_roll[:n_corr].cpu().numpy(), cu, ocfg, mask[:n_corr].cpu().numpy())
    t_corr = time.perf_counter() - t
    per_tok = t_lp / done + t_corr / n_corr
    # the same oracle pinned to one BLAS thread, on a smaller sample
    one = None
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        blas = ",".join(sorted({f"{d.get('internal_api')}({d.get('num_threads')})" for d in threadpool_info()
                                if d.get("user_api") == "blas"}))
        with threadpool_limits(limits=1, user_api="blas"):
            r = rows[:32]
            t = time.perf_counter()
            logprob_entropy(Hh[r], Wc, ids.cpu()[r], row_chunk=32)
            one = 32 / (time.perf_counter() - t)
    except Exception:
        blas = "unknown"
    return ({"value": 1.0 / per_tok, "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
             "sample": f"fp64 numpy oracle: logprob+entropy on {done} random rows of the {cfg.name} batch "
                       f"({t_lp:.1f} s) + correction (tis-srs-k3) on {n_corr} tokens ({t_corr:.1f} s); "
                       f"host {os.cpu_count()} logical cpus; BLAS {blas}",
             "logprob_tokens_per_s_1_thread": one}, dmax)


def run_reference(args):
    """--impl reference: the fp64 CPU oracle (this tier's reference arm) on the host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    import math

    import numpy as np

    from oracle import correct as oc
    from oracle.logprob import logprob_entropy

    cfg = synth.CONFIGS[args.config]
    W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed)
    n_s = 32
    ocfg = oc.Cfg(tis=True, tis_cap=2.0, log_tis_cap=math.log(2.0), seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM,
                  tau_seq=1e-3)

    def step(k):
        ids = synth.token_ids(n_s, cfg.vocab, cfg.seed + k)
        H = synth.hidden_states(n_s, cfg.hidden, cfg.seed + k, weight=W, ids=ids, mode="peaked")
        t = time.perf_counter()
        lp, _ = logprob_entropy(H, W, ids, row_chunk=32)
        roll = lp + np.random.default_rng(k).laplace(0, 2e-3, n_s)
        oc.correct(lp.astype(np.float32), roll.astype(np.float32), np.array([0, n_s]), ocfg)
        return time.perf_counter() - t

    for k in range(args.warmup):
        step(k)
    tot = sum(step(args.warmup + k) for k in range(args.steps))
    v = n_s * args.steps / tot
    out = {"impl": "reference", "metric": "logprob tokens/sec at V=151936 (1/2/4/8 B200); max |dlogp| across batch shapes",
           "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (synth/)",
           "config": {"workload": f"{cfg.name}: d={cfg.hidden}, V={cfg.vocab}; {n_s}-token sample per step",
                      "hidden": cfg.hidden, "vocab": cfg.vocab},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": _blas_threads(), "kind": "oracle",
                            "sample": f"{n_s} tokens per step through the fp64 oracle (logprob + entropy + "
                                      f"tis-srs-k3 correction)"},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "toy"],
                    help="BASELINE.json config; default c2, the largest single-GPU config")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's global batch sharded over the GPUs (default); weak: a "
                         "config-sized batch per GPU")
    ap.add_argument("--no-extra-configs", dest="extra_configs", action="store_false",
                    help="N = 1: skip the c1 / c3 extra lines")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2-persist-mb", type=int, default=-1,
                    help="device persisting-L2 set-aside in MB for our arm (-1: leave the driver default; "
                         "48 slowed the correction / PPO passes by 27%%, profiles/r02_c2_bimodal.txt)")
    ap.add_argument("--correction-tokens", type=int, default=1 << 27,
                    help="standalone correction-kernel HBM roofline at this many tokens (0 = skip)")
    ap.add_argument("--tuning", default=None,
                    help="h_policy,w_policy,sleep,slack[,group] (experiments; results unchanged)")
    ap.add_argument("--max-pairs", type=int, default=0, help="cap the persistent grid (experiments)")
    ap.add_argument("--n-seq", type=int, default=0, help="override the number of sequences (experiments)")
    ap.add_argument("--cluster-pairs", type=int, default=0, help="1 or 2 CTA pairs per cluster (experiments)")
    ap.add_argument("--no-backward-bench", dest="backward_bench", action="store_false",
                    help="skip the NEXT-3 head-backward timing")
    ap.add_argument("--no-sample-bench", dest="sample_bench", action="store_false",
                    help="skip the rollout-side twin (tim_sample) measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
