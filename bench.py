"""Headline benchmark: GLM-130B-shaped INT4 (W4A16) autoregressive decode, batch 1.

A "step" is one greedy decode step of one token through all 70 layers + the tied head
(BASELINE.json configs[3] at t = N, the only configuration its metric is quoted on).
Weights are random-init of the GLM-130B shape, generated and quantized on the GPU with the
counter-based generator, per-output-channel absmax INT4 (north_star).

Timed regions (CUDA events on the model's stream, max over ranks):
  value  : K graph replays of the decode step, state resident in HBM (63.4 GB/t of INT4
           weights per step >> 126 MB L2, so no flush is needed)
  e2e    : K calls of glm_model_decode_step (the public C ABI): pinned H2D of the token +
           position, graph replay, D2H of the greedy token, host-synchronised
  roofline: the W4A16 GEMV launches of one step replayed alone, algorithmic bytes
           (codes + fp32 scales + fp16 activations + fp32 partials) / their event time

`--impl reference` times the reference's own CPU path: oracle/_ref, the reference's unmodified
sources built with the test-infrastructure stand-ins (oracle/build_ref.sh; the Eigen product on
OpenBLAS dgemm with all host threads): one decode token through one GLM-130B-shaped layer per
step, extrapolated to 70 layers + the tied head (the oracle port when _ref is not built).
The same measurement, bounded to a few steps, is the `cpu_baseline` of the B200 line.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

G = dict(num_layers=70, hidden=12288, num_heads=96, ffn_hidden=32768, vocab=150528)
METRIC = "GLM-130B INT4 decode tokens/s (batch 1)"
PROMPT = 127  # P = 127 + [gMASK] + [sop]
SETTLE = 48   # extra untimed decode steps before the timed replays (clock settle)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """SM clock + throttle reasons DURING the timed region (B200_PROFILING.md clocks line):
    NVML every 10 ms (nvidia_ml_py), nvidia-smi every 200 ms if NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.samples, self.reasons, self.maxc = [], set(), None
        self.index = index
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.maxc = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        while not self._stop.is_set():
            self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            for n, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(n)
            self._stop.wait(0.01)

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip().split(", ")
                self.samples.append(float(out[0]))
                self.maxc = float(out[1])
                for n, v in zip(names, out[2:]):
                    if v.strip() == "Active":
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.maxc,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def self_launch(args):
    """`python bench.py --gpus N` outside torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and exit with their status; rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------------------
# CPU baseline (oracle port of the reference path) — checker infrastructure, not product
# ---------------------------------------------------------------------------------------
def cpu_layer_setup(bits=4, axis="column", seed=1):
    from oracle import pyoracle as O
    d, f = G["hidden"], G["ffn_hidden"]
    L = G["num_layers"]
    fac = (2.0 * L) ** -0.5
    xs = lambda a, b: (2.0 / (a + b)) ** 0.5
    mats = [
        O.gen_quantize(seed, 0, d, 3 * d, bits, axis, 0.0052, xs(d, d) * fac, 2 * d),
        O.gen_quantize(seed, 1, d, d, bits, axis, xs(d, d) * fac),
        O.gen_quantize(seed, 2, d, f, bits, axis, xs(d, f) * fac),
        O.gen_quantize(seed, 3, d, f, bits, axis, xs(d, f) * fac),
        O.gen_quantize(seed, 4, f, d, bits, axis, xs(f, d) * fac),
    ]
    return mats


def cpu_layer_step(mats, x):
    """One GLM-130B layer for one token: the 5 quantized linears (x . dequantize(q)) in f64."""
    import numpy as np
    from oracle import pyoracle as O
    qkv = O.qlinear_full(x, mats[0])
    a = O.qlinear_full(qkv[:, :G["hidden"]], mats[1])
    u = O.qlinear_full(a, mats[2])
    v = O.qlinear_full(a, mats[3])
    g = O.gelu(u) * v
    return O.qlinear_full(g, mats[4]), np.abs(qkv).max()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(steps, warmup):
    """The reference's CPU path timed on this host: oracle/_ref (the reference's own sources,
    oracle/build_ref.sh) when built, else the oracle port."""
    try:
        from oracle import pyref as R
        if R.available():
            return cpu_baseline_reference(R, steps, warmup)
    except Exception as e:  # noqa: BLE001 - reported in the sample text of the port baseline
        print(f"bench.py: reference CPU baseline unavailable ({e}); timing the oracle port", file=sys.stderr)
    return cpu_baseline_port(steps, warmup)


def cpu_baseline_reference(R, steps, warmup):
    threads = os.cpu_count() or 1
    head_rows = 16384
    layer_s, setup_s, head_slice_s = R.bench_layer_decode(seed=2210, bits=4, axis="column", ctx=PROMPT + 3,
                                                          warmup=warmup, steps=steps, threads=threads,
                                                          head_vocab=head_rows)
    head_s = head_slice_s * G["vocab"] / head_rows
    token_s = G["num_layers"] * layer_s + head_s
    return {
        "value": 1.0 / token_s, "unit": "tokens/s", "cores": threads, "kind": "reference",
        "sample": (f"the reference's own sources (oracle/_ref: tensor/quant/model.cpp unmodified, Eigen stand-in "
                   f"product on OpenBLAS dgemm with {threads} threads, {cpu_model()}): one decode token through one "
                   f"GLM-130B-shaped layer per step (INT4 kColumn weights through quantize_absmax + dequantize, "
                   f"matmul / attention over {PROMPT + 3} rows / deepnorm_residual / geglu, model.cpp:198-224), "
                   f"mean of {steps} after {warmup} warm-up = {layer_s:.3f} s/layer; x70 layers + the tied head "
                   f"matmul(h, transpose(E)) timed on {head_rows} of {G['vocab']} rows ({head_slice_s:.2f} s) and scaled "
                   f"linearly; setup {setup_s:.0f} s; no KV cache exists in the reference, the harness reuses the "
                   f"earlier rows' q/k/v"),
        "seconds_per_token": token_s,
    }


def cpu_baseline_port(steps, warmup):
    import numpy as np
    t0 = time.time()
    mats = cpu_layer_setup()
    setup_s = time.time() - t0
    x = np.random.default_rng(0).normal(size=(1, G["hidden"]))
    for _ in range(warmup):
        cpu_layer_step(mats, x)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        cpu_layer_step(mats, x)
        times.append(time.perf_counter() - t)
    layer_s = statistics.median(times)
    d, f, V = G["hidden"], G["ffn_hidden"], G["vocab"]
    layer_macs = d * 3 * d + d * d + 2 * d * f + f * d
    head_s = layer_s * (V * d) / layer_macs  # bf16 head GEMV, same per-MAC cost (labelled)
    token_s = G["num_layers"] * layer_s + head_s
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {
        "value": 1.0 / token_s, "unit": "tokens/s", "cores": threads, "kind": "port",
        "sample": (f"oracle port ({cpu_model()}): one GLM-130B layer decode (5 INT4 per-output-channel linears, x . dequantize(q) in f64, "
                   f"oracle port of quant.cpp:188-221 + tensor.cpp:135-155) per step, median of {steps} after "
                   f"{warmup} warm-up; extrapolated x70 layers + head by MACs; {layer_s:.2f} s/layer; "
                   f"setup {setup_s:.0f} s (gen+quantize one layer)"),
        "seconds_per_token": token_s,
    }


DTYPE = "int4 x s16 (u8 x s8 IMMA digits, int32 accumulate)"


def workload_config(B, world, warmup):
    """The workload both arms report (BASELINE configs[3] at batch B on `world` GPUs)."""
    return {"workload": "GLM-130B-shaped 70-layer INT4 decode (BASELINE configs[3]): hidden 12288, 96 heads, "
                        "ffn 32768 (GeGLU), vocab 150528, random-init counter-based weights (model.cpp:69-104 stds), "
                        "absmax INT4 per output channel (kColumn)",
            "global_batch": B, "seq_len": PROMPT + 2, "context_at_timing": PROMPT + 2 + 3 + warmup + SETTLE,
            "parallelism": f"tp{world}", "l2": "inputs larger than L2 (63.4 GB of weights over the ranks)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cb = cpu_baseline(args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds_per_token"] * 1000.0,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(1, args.gpus, args.warmup),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------------
def gemv_traffic():
    """Per-launch DRAM bytes (read + write) of the GEMV, averaged over the four GEMV launches
    of one layer, from the committed `ncu --set full` capture (profiles/gemv_traffic.json)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "gemv_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def gemv_bytes_per_step(m_rows, t):
    """Algorithmic bytes of the W4A16 GEMV launches of one decode step on one rank."""
    d, f, L = G["hidden"], G["ffn_hidden"], G["num_layers"]
    shapes = [(d, 3 * d // t), (d // t, d), (d, 2 * f // t), (f // t, d)]  # qkv, out, w1|v fused, w2
    total = 0
    for K, N in shapes:
        total += K * N // 2 + N * 4 + m_rows * K * 2 + m_rows * N * 4
    return total * L


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2210_02414_b200 import glm

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = args.batch
    cfg = glm.GLMConfig(**G)
    max_ctx = PROMPT + 2 + args.warmup + SETTLE + args.steps + args.e2e_steps + 8
    t0 = time.time()
    m = glm.Model(cfg, bits=4, axis="column", max_batch=B, max_ctx=max_ctx, head_bf16=True, tp_rank=rank,
                  tp_size=world)
    if world > 1:
        uid = [glm.tp_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        m.init_comm(uid[0])
    m.init_synthetic(args.seed)
    init_s = time.time() - t0
    rng = np.random.default_rng(1234)
    prompt = [int(v) for v in rng.integers(6, 150000, size=PROMPT)]
    positions, C = glm.gmask_layout(PROMPT, 0)
    for b in range(B):
        m.prefill(prompt + [2], positions[:C], C, seq=b, logits=False)
    # three warm-up steps through the public API (host token ids in / out)
    tok = [3] * B
    pos = [PROMPT] * B
    for _ in range(3):
        nxt, _ = m.decode_step(tok, pos)
        tok, pos = [int(v) for v in nxt], [p + 1 for p in pos]
    # device-timed K steps (graph replays), clocks sampled during the region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # clock settle: the timed replays start after >= SETTLE untimed steps on top of --warmup
    # (the power-capped SM clock takes a few hundred ms to reach its steady state)
    with ClockSampler(local) as clk:
        ms, gemv_ms, launches = m.bench_decode(B, args.steps, args.warmup + SETTLE)
    torch.cuda.synchronize()
    if world > 1:
        mt = torch.tensor([ms, gemv_ms], device="cuda")
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms, gemv_ms = (float(v) for v in mt.tolist())
    # e2e through the public API right after, at the same settled clocks: host token ids in,
    # next token ids out (pinned H2D / D2H inside every step); the replays advanced the caches
    pos = [p + args.warmup + SETTLE + args.steps for p in pos]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(args.e2e_steps):
        nxt, _ = m.decode_step(tok, pos, logits=False)
        tok, pos = [int(v) for v in nxt], [p + 1 for p in pos]
    e2e_s = time.perf_counter() - t
    if world > 1:
        e2e_t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_t.item())
    e2e_tps = B * args.e2e_steps / e2e_s
    mem = m.memory()
    if rank != 0:
        return
    pk = peaks()
    hbm = pk["hbm_gbs"]
    gb = gemv_bytes_per_step(B, world)
    achieved = gb / (gemv_ms * 1e-3) / 1e9
    value = B * 1000.0 / ms
    weights_per_rank = mem["quant_payload_bytes"] / world
    roofline_step_ms = weights_per_rank / (hbm * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPE, "data": "synthetic",
        "precision": "W4A16: int4 weight codes x fp16 activations re-expressed as exact 16-bit fixed-point digits on "
                     "the integer MMA (int32 accumulation); fp32 residual / LayerNorm; bf16 tied head",
        "config": dict(workload_config(B, world, args.warmup), frac_of_weight_roofline=roofline_step_ms / ms),
        "e2e": {"value": e2e_tps, "unit": "tokens/s", "h2d_bytes_per_step": 8 * B, "d2h_bytes_per_step": 4 * B,
                "steps": args.e2e_steps},
        "gpu_launches": launches * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": gemv_traffic(), "kernel": "k_gemv_i4 (W4A16 GEMV on the integer MMA, 280 launches/step)",
                     "algorithmic_bytes_per_step": gb, "gemv_ms_per_step": gemv_ms,
                     "gemv_share_of_step": gemv_ms / ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in pk else "fallback 6650"},
        # north_star's step-level metric: INT4 weight bytes per step / aggregate HBM bandwidth
        "weight_roofline": {"frac": roofline_step_ms / ms, "ideal_ms_per_step": roofline_step_ms,
                            "weight_bytes_per_rank": weights_per_rank, "peak_gbs": hbm},
        "clocks": clk.summary(),
        "init_seconds": init_s,
    }
    if not args.no_cpu_baseline and world == 1:
        del m  # the CPU baseline needs ~40 GB of host memory; the model's device state is done
        cb = cpu_baseline(max(1, min(3, args.steps)), 1)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--seed", type=int, default=2210)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
