#!/usr/bin/env python
"""bench.py -- per-round hot path of batch speculative decoding on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen3|vicuna|glm4|toy]
                    [--impl ours|reference]

A step is one EqSpec verification round over one batch:
specdec_verify (K1) -> specdec_rebuild_pos_mask (K3) -> specdec_realign_kv (K2, in
place), on one stream, no host synchronisation.  Default workload: the Qwen3-8B-shaped
KV (36 layers x 8 KV heads x 128, bf16), B=8, k=5, vocab 151936, contexts
n_i ~ U[1536, 2048] (BASELINE.json north_star target config), alpha_i ~ U[0.5, 0.9].

Inputs are synthetic (synth/): planted logits ring (16 buffers, > L2) + matching drafts,
hashed KV over the full capacity.  `value` = rounds/s with inputs resident in HBM;
`e2e` = the same rounds through the C ABI with each step's logits + drafts copied from
pinned host memory and the step's (accept, bonus, emit) read back.  `--impl reference`
times the CPU oracle (oracle/) on the same workload.  N > 1 runs independent replicas
(one process per GPU; the EqSpec round does not shard -- DESIGN.md "Multi-GPU").
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import workloads as W  # noqa: E402

METRIC = "verify+realign rounds/s (B=8,k=5); KV-realign HBM GB/s vs ~8 TB/s peak"
RING = 16


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="qwen3", choices=["qwen3", "vicuna", "glm4", "toy", "pool"])
    ap.add_argument("--pool-n", type=int, default=1024, help="pool: total sequences (all ranks)")
    ap.add_argument("--pool-lengths", default="random", choices=["random", "uniform"])
    ap.add_argument("--pool-W", type=int, default=0, help="pool: window (0 = whole shard, <= 2048)")
    ap.add_argument("--min-group", type=int, default=2)
    ap.add_argument("--max-new", type=int, default=256)
    ap.add_argument("--shard", default="balanced", choices=["band", "strided", "balanced"],
                    help="pool sharding over ranks: equal-count bands, strided, or bands of "
                         "equal estimated cost (prompt length + max_new per sequence)")
    ap.add_argument("--pool-consumer", default="zero-copy", choices=["zero-copy", "dense", "slot"],
                    help="pool: same-length batches run on the pool slots (zero-copy) or are "
                         "gathered into a dense staging rectangle too (PAPER.md:537); slot: a "
                         "slot-indexed consumer, no batch moves KV (SURVEY 8f f3)")
    ap.add_argument("--pool-exec", default="native", choices=["native", "python"],
                    help="pool: per-batch launch loop in C++ (specdec_pool_epoch) or Python")
    ap.add_argument("--alg3-graph", type=int, default=1,
                    help="pool --pool-mode alg3: replay the device loop from a CUDA graph of 16 iterations (0: direct, "
                         "2: the KV moves in conditional graph nodes)")
    ap.add_argument("--pool-scatter-stream", type=int, default=1,
                    help="pool (native, overlapped): the scatters on a third stream beside the gathers")
    ap.add_argument("--pool-verify-group", type=int, default=64,
                    help="pool (native executor): same-length batches verified per launch (1 = per batch)")
    ap.add_argument("--pool-staging", type=int, default=2,
                    help="pool, native executor: staging buffers; >= 2 overlaps the fallback "
                         "gathers (copy stream) with the same-length batches, 1 = serial")
    ap.add_argument("--pool-est", type=float, nargs=2, default=(0.0, 0.0), metavar=("GBPS", "VERIFY_US"),
                    help="pool, overlapped executor: scheduling estimates (0 = library defaults)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="pool, 1 GPU: drain each of G band shards alone and report the predicted "
                         "G-GPU throughput (slowest shard); a prediction, not a measurement")
    ap.add_argument("--shard-c", type=float, default=1.0,
                    help="--shard balanced: per-sequence weight = prompt length + c * max_new")
    ap.add_argument("--pool-patience", type=int, default=2,
                    help="pool epoch plan: leftovers wait up to P epochs for a same-length partner before "
                         "a fallback batch (reading R27, specdec_pool_group_deferred); 0 = R11's full plan "
                         "(N=1024: 3003 seq/s at P=0, 7428 at P=2)")
    ap.add_argument("--pool-pipeline", type=int, default=0,
                    help="pool epoch mode, native executor: a plan's mixed batches run on the copy stream beside "
                         "the next plan, which leaves their members out (reading R28)")
    ap.add_argument("--pool-mode", default="epoch", choices=["epoch", "alg3"],
                    help="epoch: run every batch of the window plan; alg3: batch 0 then re-plan")
    ap.add_argument("--B", type=int, default=0, help="override batch size")
    ap.add_argument("--pattern", default="alpha", choices=list(W.ACCEPT_PATTERNS))
    ap.add_argument("--alpha", type=float, default=0.7, help="acceptance rate of --pattern fixed")
    ap.add_argument("--ctx", type=int, default=0, help="override the context: n ~ U[ctx-512, ctx]")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1,
                    help="repeat the timed region (value) this many times and report the median")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--episode", type=int, default=32,
                    help="restore the initial lengths every N rounds (stationary workload; 0 = never)")
    ap.add_argument("--anchor", action="store_true",
                    help="f3: anchored-origin realign (K1 moves the KV origin to minimise moved rows)")
    ap.add_argument("--draft-kv", action="store_true",
                    help="f1: the draft model keeps its own KV cache, realigned every round too")
    ap.add_argument("--kv-mode", default="inplace", choices=["inplace", "pingpong"],
                    help="K2 in place, or out of place between two KV buffers (copies Delta=0 rows too)")
    ap.add_argument("--round-mode", default="graph-block",
                    choices=["graph-block", "graph-fork", "graph-serial", "direct-fork", "direct-serial"],
                    help="value region: CUDA graphs of one episode of rounds (block), one graph per "
                         "round, or direct launches; K3 forked under K2 or serial")
    return ap.parse_args(argv)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_ burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def coll_device(device):
    """Tensors for collectives live on the GPU under NCCL, on the host under gloo."""
    import torch
    import torch.distributed as dist
    return device if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float, device, world: int) -> float:
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(config_key):
    """dram bytes per launch of K2 from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p)).get(config_key)
    if not d:
        return None, None
    return d["realign_dram_bytes_per_launch"], (
        f"ncu --set full capture of one K2 launch: {d['realign_dram_bytes_per_launch'] / 1e9:.3f} GB DRAM "
        f"vs {d['algorithmic_bytes_same_launch'] / 1e9:.3f} GB algorithmic for that launch "
        f"(ratio {d['traffic_over_algorithmic']}); {d['source']}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML samples of SM clock and throttle reasons while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- clocks are reported as unavailable
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
def shape_for(args):
    sh = W.SHAPES[args.config]
    if args.B:
        sh = sh.with_(B=args.B)
    if args.ctx:   # SURVEY §8d ctx sweep: n ~ U[ctx - 512, ctx]
        sh = sh.with_(ctx=args.ctx, len_lo=max(1, args.ctx - 512), len_hi=args.ctx)
    return sh


# draft models of the BASELINE pairs (layers, KV heads, head_dim): Vicuna-68M (2 x 12 x 64),
# Qwen3-0.6B (28 x 8 x 128) for the Qwen3 and GLM-4 pairs; toy drafter = toy shape.
DRAFT_DIMS = {"vicuna": (2, 12, 64), "qwen3": (28, 8, 128), "glm4": (28, 8, 128), "toy": (2, 2, 8)}


def workload_name(sh, args):
    d = f", draft KV {DRAFT_DIMS[sh.name]} realigned too" if getattr(args, "draft_kv", False) else ""
    d += ", anchored origin (f3)" if getattr(args, "anchor", False) else ""
    d += ", ping-pong KV (out of place)" if getattr(args, "kv_mode", "inplace") == "pingpong" else ""
    return (f"{sh.name} EqSpec round: B={sh.B} k={sh.k} V={sh.V} KV {sh.layers}x{sh.H}x{sh.D} "
            f"{sh.kv_dtype}, n~U[{sh.len_lo},{sh.len_hi}], accept={args.pattern}"
            f"{f' alpha={args.alpha}' if args.pattern == 'fixed' else ''}{d}")


class RoundBench:
    """Device state + logits/draft ring for the timed EqSpec rounds."""

    def __init__(self, sh, args, device, total_rounds):
        import torch

        from paper_2510_22876_b200.eqspec import EqSpecBatch
        self.torch = torch
        self.sh, self.dev = sh, device
        B, k = sh.B, sh.k
        self.cap = W.derive_cap(sh, total_rounds) if sh.name != "toy" else max(sh.cap, W.derive_cap(sh, total_rounds))
        self.lengths = W.gen_lengths(sh, args.seed, B)
        self.tokens = W.left_padded_tokens(self.lengths, self.cap, args.seed, sh.V)
        draft = DRAFT_DIMS[sh.name] if args.draft_kv else None
        # f3: slack for the moving origin: at most k+1 columns of drift per round
        slack = (k + 1) * total_rounds if args.anchor else 0
        self.bt = EqSpecBatch(B, k, self.cap, sh.layers, sh.H, sh.D, sh.kv_dtype, device, draft=draft,
                              anchor_slack=slack, kv_mode=args.kv_mode)
        # ping-pong: the method's (algorithmic) KV bytes are those of the rows that shift;
        # K2 also copies the Delta = 0 rows (counted by the device `moved` counter)
        self.alg_rows = torch.zeros(1, dtype=torch.int64, device=device)
        # kept KV rows of every round (region B): the moved share = moved / all kept bytes
        self.kept_rows = torch.zeros(1, dtype=torch.int64, device=device)
        if draft is not None:
            self.bt.dkv.copy_(W.gen_kv_torch(args.seed + 1, self.bt.dkv.shape, self.bt.dkv.dtype, device))
        self.bt.load(self.tokens, self.lengths)
        self.bt.kv.copy_(W.gen_kv_torch(args.seed, self.bt.kv.shape, self.bt.kv.dtype, device))
        self.logits = [W.gen_logits_torch(args.seed, r, B, k, sh.V, sh.logit_dtype, device)
                       for r in range(RING)]
        self.truth = [W.gen_round_truth(args.seed, r, B, k, sh.V, args.pattern, alpha=args.alpha) for r in range(RING)]
        self.drafts = [torch.from_numpy(t.draft).to(device) for t in self.truth]
        self.stream = torch.cuda.current_stream(device)

    def reset(self):
        self.bt.load(self.tokens, self.lengths)   # KV content is arbitrary; (n, p) restart
        bt = self.bt
        if not hasattr(self, "snap"):
            self.snap = (bt.tok[0].clone(), bt.n[0].clone(), bt.pad[0].clone())

    def reset_fast(self):
        """Episode boundary: restore the initial (tokens, n, p) state with device copies on
        the stream (no host sync), so every timed round sees the same ctx ~2048 workload
        whatever --steps is.  KV bytes are arbitrary synthetic data either way."""
        bt = self.bt
        bt.tok[0].copy_(self.snap[0], non_blocking=True)
        bt.n[0].copy_(self.snap[1], non_blocking=True)
        bt.pad[0].copy_(self.snap[2], non_blocking=True)
        bt.active.fill_(1)
        if bt.anchor is not None:
            bt.anchor.fill_(bt.anchor_slack)
        bt.cur = 0

    def capture_block(self, episode_len, hook=None):
        """One CUDA graph per episode: the episode's state reset (3 device copies) and its
        `episode_len` rounds (ring slot r % RING, parity alternating; an even count, so the
        graph ends at the parity it starts from).  `hook(r, stream)`, if given, is captured
        after round r (tests: snapshots of the per-round results); the bench passes none."""
        import torch
        bt = self.bt
        self.reset()
        cs = torch.cuda.Stream(self.dev)
        cs.wait_stream(self.stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
            self.reset_fast()
            for r in range(episode_len):
                bt.launch_round(self.logits[r % RING], self.drafts[r % RING], stream=cs)
                if hook is not None:
                    hook(r, cs)
                bt.cur = 1 - bt.cur
        self.stream.wait_stream(cs)
        torch.cuda.synchronize()
        return g

    def episode(self, r, episode_len):
        if episode_len and r and r % episode_len == 0:
            self.reset_fast()

    def step(self, r, ev=None):
        import torch
        bt, lg, d = self.bt, self.logits[r % RING], self.drafts[r % RING]
        if ev is not None:
            # keep the GPU busy while Python enqueues this round, so that the event
            # intervals hold kernel time only (short rounds: no host launch gaps)
            with torch.cuda.stream(self.stream):
                torch.cuda._sleep(SLEEP_CYCLES)
            ev[0].record(self.stream)
        bt.verify(lg, d)
        if ev is not None:
            ev[1].record(self.stream)
        bt.repad(d)
        if ev is not None:
            ev[2].record(self.stream)
        bt.realign()
        if ev is not None:
            ev[3].record(self.stream)
            self.kept_rows += bt.kept.long().sum()
            if bt.kv_mode == "pingpong":
                c = bt.cur
                self.alg_rows += (bt.kept.long() * (bt.pad[c] != bt.pad[1 - c])).sum()
        bt.cur = 1 - bt.cur

    def mean_width(self):
        return None


def run_ours(args, rank, world, device):
    """Three timed regions, each bracketed by barrier + synchronize:
      A  `value`: K rounds replayed from CUDA graphs (one graph per (parity, ring slot)),
         inputs resident in HBM;
      B  kernel timing: the same K rounds launched directly with CUDA events around each
         kernel on the launching stream -> per-kernel durations for the roofline;
      C  `e2e`: K rounds whose logits + drafts are copied from pinned host memory (copy
         stream, double-buffered) and whose (accept, bonus, emit) are read back.
    The state (n, p, tokens) is reset before each region so all three see the same work."""
    import torch
    import torch.distributed as dist

    sh = shape_for(args)
    total = args.warmup + args.steps + 2
    rb = RoundBench(sh, args, device, total)
    bt = rb.bt
    torch.cuda.synchronize()
    launch_bytes = []
    for r in range(args.warmup):          # direct launches: sets kernel attributes
        m0 = int(bt.moved.item())
        rb.step(r)
        launch_bytes.append(int(bt.moved.item()) - m0)   # K2 bytes of this launch
    torch.cuda.synchronize()
    log = os.environ.get("SPECDEC_BENCH_LAUNCH_LOG")
    if log:   # per-launch algorithmic K2 bytes of the first warm-up launches (for ncu)
        with open(log, "w") as f:
            json.dump({"config": f"{sh.name}_B{sh.B}", "realign_bytes_per_launch": launch_bytes}, f)
    bt.fork = args.round_mode.endswith("fork")
    use_graph = args.round_mode.startswith("graph")
    bt.V = sh.V
    if use_graph:
        bt.capture(list(zip(rb.logits, rb.drafts)), V=sh.V)
    # graph-block: one CUDA graph per episode -- the episode's state reset (3 device copies)
    # and its `episode` rounds (ring slot r % RING, parity alternating; an even count, so the
    # graph ends at the parity it starts from) -- so short rounds are not bound by one host
    # replay call each.  Same kernels, same order, same bytes as the per-round graphs.
    block = None
    blk = args.episode
    tails = {}
    if args.round_mode == "graph-block" and blk and blk % RING == 0 and blk % 2 == 0:
        block = rb.capture_block(blk)
        # the rounds after the last whole episode (e.g. a 20-step run) replay a block graph
        # of their own: the episode's reset + those rounds (captured here, outside timing)
        for m in {args.steps % blk, args.warmup % blk} - {0}:
            tails[m] = rb.capture_block(m)

    def one_round(r):
        if use_graph:
            bt.replay(r % RING)
        else:
            bt.launch_round(rb.logits[r % RING], rb.drafts[r % RING])
            bt.cur = 1 - bt.cur

    def run_rounds(n):
        r = 0
        if block is not None:
            while r + blk <= n:
                block.replay()           # reset + blk rounds; bt.cur is back where it started
                bt._last = 1 - bt.cur
                r += blk
            if n - r in tails:           # reset + the remaining rounds (parities 0, 1, ...)
                tails[n - r].replay()
                bt.cur, bt._last = (n - r) % 2, (n - r - 1) % 2
                r = n
        for q in range(r, n):
            rb.episode(q, args.episode)
            one_round(q)

    def sync():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- A: value (graphs); --reps R: R timed repetitions, the median is reported
    rb.reset()
    run_rounds(args.warmup)
    clocks = ClockSampler(device.index if device.index is not None else 0)
    reps = []
    with clocks:
        for _ in range(max(1, args.reps)):
            rb.reset()
            moved0 = int(bt.moved.item())
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            sync()
            t0.record(rb.stream)
            run_rounds(args.steps)
            t1.record(rb.stream)
            torch.cuda.synchronize()
            sync()
            reps.append(max_over_ranks(t0.elapsed_time(t1), device, world))
            moved_A = int(bt.moved.item()) - moved0
    ms = float(np.median(reps))
    width_end = int((bt.pad_cur + bt.n_cur).max().item())
    status = int(bt.status.item())
    # ---- B: per-kernel events (direct launches, same rounds)
    rb.reset()
    moved0 = int(bt.moved.item())
    rb.kept_rows.zero_()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    # the moved-bytes counter after every round (a device copy on the launching stream,
    # outside the event intervals): per-launch K2 bytes for the per-launch rate spread
    snap = torch.zeros(args.steps + 1, dtype=torch.int64, device=device)
    sync()
    with torch.cuda.stream(rb.stream):
        snap[0].copy_(bt.moved[0])
    for r in range(args.steps):
        rb.episode(r, args.episode)
        rb.step(r, evs[r])
        with torch.cuda.stream(rb.stream):
            snap[r + 1].copy_(bt.moved[0])
    sync()
    moved_B = int(bt.moved.item()) - moved0
    per_launch = np.diff(snap.cpu().numpy())
    # algorithmic K2 bytes of region B: in place = the device counter (only shifting rows
    # move); ping-pong = the shifting rows' bytes, although every kept row is copied
    alg_B = moved_B if bt.kv_mode == "inplace" else int(rb.alg_rows.item()) * 2 * sh.bpt
    k1 = sum(e[0].elapsed_time(e[1]) for e in evs)
    k3 = sum(e[1].elapsed_time(e[2]) for e in evs)
    k2 = sum(e[2].elapsed_time(e[3]) for e in evs)
    # ---- C: e2e
    e2e = None if args.no_e2e else run_e2e(rb, args, world)
    logits_bytes = sh.B * (sh.k + 1) * sh.V * (4 if sh.logit_dtype == "fp32" else 2)
    kept_bytes = 2 * int(rb.kept_rows.item()) * sh.bpt
    k2_each = np.array([e[2].elapsed_time(e[3]) for e in evs])
    return dict(sh=sh, ms=ms, reps_ms=reps, moved=alg_B, copied=moved_B, moved_A=moved_A, kept_bytes=kept_bytes,
                k2_launches=(per_launch, k2_each),
                k1_ms=k1, k3_ms=k3,
                kernels_per_round=bt.kernels_per_round,
                k2_ms=k2, status=status | int(bt.status.item()), clocks=clocks.summary(), e2e=e2e,
                end_width=width_end, logits_bytes=logits_bytes)


def k2_spread(nbytes, ms, peak):
    """Per-launch K2 rates over the kernel-timing region: how the launch-level rate depends on
    the bytes a launch moves (small launches: the fixed launch / first-load / last-store cost
    weighs more), and the time share of launches that move nothing."""
    nbytes, ms = np.asarray(nbytes, np.float64), np.asarray(ms, np.float64)
    mv = nbytes > 0
    if not mv.any():
        return None
    rate = nbytes[mv] / (ms[mv] / 1e3) / 1e9
    q = lambda x: [float(v) for v in np.percentile(x, [0, 25, 50, 75, 100])]
    # least squares t = t0 + bytes / R over the moving launches: t0 = fixed cost per launch,
    # R = the streaming rate once the stream is full
    A = np.stack([np.ones(mv.sum()), nbytes[mv]], 1)
    (t0, inv), *_ = np.linalg.lstsq(A, ms[mv] / 1e3, rcond=None)
    return {"launches": int(len(ms)), "zero_byte_launches": int((~mv).sum()),
            "zero_byte_time_share": float(ms[~mv].sum() / ms.sum()) if ms.sum() else 0.0,
            "MB_quartiles": [x / 1e6 for x in q(nbytes[mv])], "GBps_quartiles": q(rate),
            "fit_fixed_us": float(t0 * 1e6), "fit_stream_GBps": float(1 / inv / 1e9) if inv > 0 else None,
            "fit_stream_frac": float(1 / inv / 1e9 / peak) if inv > 0 else None}


def round_bandwidth(res, sh, args, peak):
    k2 = res["moved_A"] / args.steps if args.kv_mode == "inplace" else res["moved"] / args.steps
    width = res["end_width"]
    k3 = sh.B * width * 8 * 2 + 2 * sh.B * (width + sh.k) * 8     # tokens read + written, mask + pos
    tot = res["logits_bytes"] + k2 + k3
    gbps = tot / (res["ms"] / args.steps / 1e3) / 1e9
    return {"bytes_per_round": tot, "GBps": gbps, "frac": gbps / peak,
            "note": "K1 logits + K2 algorithmic KV bytes + K3 token/mask/pos bytes per round, over the "
                    "value region's round time (K1/K3 latency included)"}


def run_e2e(rb, args, world):
    """End to end through the C ABI with HOST buffers: every step is one
    specdec_eqspec_round_host call (eqspec.py step_host) that copies the step's logits +
    drafts from pinned host memory into a device staging slot (copy stream), runs the
    round (K1 -> K3 -> K2) on the compute stream and copies the step's result -- the
    per-row emitted-token counts -- back into pinned host memory (third stream).  Three
    staging slots and one result set per state parity let the copy of step s start two
    rounds ahead of its use (absorbing an occasional slow H2D); nothing synchronises the
    host inside the timed region."""
    import torch
    import torch.distributed as dist
    sh, dev, bt = rb.sh, rb.dev, rb.bt
    d2h_mode = os.environ.get("SPECDEC_E2E_D2H", "one")
    from paper_2510_22876_b200.eqspec import pack_host_inputs
    # each step's logits + drafts in one pinned buffer: one H2D per step
    host_lg, host_dr = zip(*[pack_host_inputs(lg, d) for lg, d in zip(rb.logits, rb.drafts)])
    out_e = torch.empty((args.steps, sh.B), dtype=torch.int32).pin_memory()
    comp = rb.stream
    bt.host_io(host_lg[0], host_dr[0])

    def run(n):
        for r in range(n):
            rb.episode(r, args.episode)
            bt.step_host(host_lg[r % RING], host_dr[r % RING],
                         None if d2h_mode == "none" else out_e[r], V=sh.V, stream=comp)
        comp.wait_stream(bt._io_streams[1])

    rb.reset()
    run(min(args.warmup, args.steps))
    torch.cuda.synchronize()
    rb.reset()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    run(args.steps)
    e1.record(comp)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = max_over_ranks(e0.elapsed_time(e1), dev, world)
    # the results are the method's: every step's emit = planted accept + 1 (no EOS/budget)
    if d2h_mode != "none":
        for r in range(args.steps):
            assert np.array_equal(out_e[r].numpy(), rb.truth[r % RING].accept + 1), "e2e emit mismatch"
    h2d_b = rb.logits[0].numel() * rb.logits[0].element_size() + rb.drafts[0].numel() * 8
    d2h_b = {"one": sh.B * 4, "none": 0}[d2h_mode]
    return {"value": world * args.steps / (ms / 1e3), "unit": "rounds/s", "h2d_bytes_per_step": h2d_b,
            "d2h_bytes_per_step": d2h_b, "ms_per_step": ms / args.steps, "wall_s": wall,
            "api": "specdec_eqspec_round_host (one C call per step: H2D + K1/K3/K2 + D2H)",
            "overlap": "H2D on a copy stream into three staging slots; round on the compute stream; "
                       "D2H on a third stream from the round's parity result set"}


# ----------------------------------------------------------------------------- oracle timing
def oracle_round_sample(sh, args, rounds=2, seed=0, threads=1):
    """Time the CPU oracle (never tuned) on the same workload: whole rounds -- Alg. 1 over
    the full logits tail, the token repad, and Realign over EVERY plane of the KV (no
    extrapolation) -- on `threads` host threads.  threads == 1 runs the serial oracle
    functions; threads > 1 the thread-parallel driver (oracle/driver.py: the same
    functions on independent batch rows and (plane, row) slab groups).  Input generation
    is outside the timed region.  Returns (rounds/s, per-part seconds per round)."""
    from oracle import align as OA
    from oracle import driver as OD
    from oracle import verify as OV
    B, k = sh.B, sh.k
    cap = W.derive_cap(sh, rounds + 2)
    lengths = W.gen_lengths(sh, seed, B)
    tokens = W.left_padded_tokens(lengths, cap, seed, sh.V)
    shp = (sh.n_planes, B, sh.H, cap, sh.D)
    kv = W.gen_kv_bits_np(seed, int(np.prod(shp))).reshape(shp)
    n = lengths.astype(np.int32)
    L = int(n.max())
    pad = (L - n).astype(np.int32)
    act = np.ones(B, np.uint8)
    ins = [(W.gen_logits_np(seed, r, B, k, sh.V, sh.logit_dtype),
            W.gen_round_truth(seed, r, B, k, sh.V, args.pattern, alpha=args.alpha)) for r in range(rounds)]
    tv = tr = tk = 0.0
    with OD.make_pool(threads) as pool:
        for bits, rt in ins:
            a = time.perf_counter()
            if threads > 1:
                v = OD.batch_verify_parallel(pool, bits, sh.logit_dtype, rt.draft, n, pad, act)
            else:
                v = OV.batch_verify(bits, sh.logit_dtype, rt.draft, n, pad, act)
            b = time.perf_counter()
            tokens, _, _ = OA.repad_tokens(tokens, cap, k, pad, L, v)
            c = time.perf_counter()
            if threads > 1:
                OD.realign_parallel(pool, kv, pad, v["pad_new"], v["kept"])
            else:
                OA.realign_kv_inplace(kv, pad, v["pad_new"], v["kept"])
            d = time.perf_counter()
            tv, tr, tk = tv + b - a, tr + c - b, tk + d - c
            n, pad, L = v["n_new"], v["pad_new"], v["L_new"]
    per_round = (tv + tr + tk) / rounds
    return 1.0 / per_round, dict(verify_s=tv / rounds, repad_s=tr / rounds, realign_s=tk / rounds,
                                 planes=sh.n_planes, rounds=rounds, threads=threads)


def round_cpu_baseline(sh, args, rounds=2):
    """cpu_baseline of the round line: the oracle on `nproc` host threads (value) and on one
    thread, both over whole rounds of the bench workload."""
    from oracle import driver as OD
    nthr = OD.host_threads()
    rps_n, parts_n = oracle_round_sample(sh, args, rounds=rounds, threads=nthr)
    rps_1, parts_1 = oracle_round_sample(sh, args, rounds=rounds, threads=1)
    return {"value": rps_n, "unit": "rounds/s", "cores": nthr, "kind": "oracle",
            "sample": (f"{rounds} whole oracle rounds of the {sh.name} workload (verify over the full "
                       f"logits tail, repad, realign over all {sh.n_planes} KV planes; no extrapolation), "
                       f"thread-parallel driver over batch rows and (plane, row) slabs on {nthr} threads "
                       f"(oracle/driver.py); numpy on {cpu_info()}"),
            "nproc": nthr, "cpu_model": cpu_info(), "parts_s": parts_n,
            "single_thread": {"value": rps_1, "cores": 1, "parts_s": parts_1}}


def cpu_info():
    model = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model


def pool_workload(args):
    """Prompt lengths (incl. the pending token) and admission order of the pool workload."""
    N = args.pool_n
    rng_h = W.hash_np(args.seed, W.S_POOL, np.arange(N))
    if args.pool_lengths == "uniform":
        lens = np.full(N, 256, np.int32)                      # All-Mean analog
    else:
        lens = (64 + (rng_h % np.uint64(512 - 64 + 1)).astype(np.int64)).astype(np.int32)
    order = np.array(sorted(range(N), key=lambda s: (int(lens[s]), s)), np.int32)  # sort on
    return lens, order


def oracle_pool_sample(args, verify_samples=2, threads=1):
    """The CPU oracle on the pool workload, as a bounded sample: the oracle's own GetBatch
    plan (oracle.pool.form_batches, timed in full) drives the whole drain with the planted
    accept lengths; the per-batch Alg. 1 verify (oracle.verify.batch_verify over the full
    B x (k+1) x V logits) and the KV gather copy rate (oracle.align.copy_rows of one whole
    member, all 72 planes) are timed on samples and extrapolated to the drain's batch count
    and algorithmic KV bytes.  threads > 1: the thread-parallel driver (oracle/driver.py:
    batch rows / planes on separate threads).  Returns (sequences/s, parts)."""
    from oracle import align as OA
    from oracle import driver as OD
    from oracle import pool as OP
    from oracle import verify as OV
    sh = W.SHAPES["qwen3"]
    k, V, B = sh.k, sh.V, sh.B
    lens, order = pool_workload(args)
    N = len(lens)
    Wn = min(args.pool_W or N, 2048, N)
    o_len, gen, act = lens.astype(np.int64), np.zeros(N, np.int64), np.ones(N, np.uint8)
    wait = np.zeros(N, np.int64)          # R27 (epoch mode with --pool-patience)
    pipe = bool(args.pool_pipeline) and args.pool_mode != "alg3"
    inflight = []                         # R28 (--pool-pipeline): the last plan's mixed members
    truth = [W.gen_round_truth(args.seed, r, B, k, V, args.pattern, alpha=args.alpha) for r in range(RING)]
    t_plan = 0.0
    n_batches = n_same = same_members = fb_members = 0
    kv_bytes = 0
    dense = args.pool_consumer == "dense"
    slot = args.pool_consumer == "slot"
    while act.any():
        t0 = time.perf_counter()
        act_plan = OP.pipeline_window_active(act, inflight) if pipe else act
        if args.pool_patience > 0 and args.pool_mode != "alg3":
            plan = OP.form_batches_deferred(o_len, act_plan, order, Wn, B, args.min_group, wait, args.pool_patience)
        else:
            plan = OP.form_batches(o_len, act_plan, order, Wn, B, args.min_group)
        t_plan += time.perf_counter() - t0
        if pipe:
            if not plan["batches"]:       # every active member in flight: they finish, then re-plan
                inflight = []
                continue
            inflight = OP.mixed_members(plan)
        nb = 1 if args.pool_mode == "alg3" else len(plan["batches"])
        for b in range(nb):
            mem = plan["batches"][b]
            if plan["kind"][b]:
                n_same += 1
                same_members += len(mem)
            else:
                fb_members += len(mem)
            acc = truth[n_batches % RING].accept
            for j, s in enumerate(mem):
                e = min(int(acc[j]) + 1, args.max_new - int(gen[s]))
                if dense or (not plan["kind"][b] and not slot):
                    kv_bytes += 2 * (int(o_len[s]) - 1) * sh.bpt + 2 * (int(acc[j]) + 1) * sh.bpt
                o_len[s] += e
                gen[s] += e
                if gen[s] >= args.max_new:
                    act[s] = 0
            n_batches += 1
    # per-batch verify, timed on samples of the same logits
    t_ver = []
    pool = OD.make_pool(threads)
    for r in range(verify_samples):
        bits = W.gen_logits_np(args.seed, r, B, k, V, sh.logit_dtype)
        n = np.full(B, 300, np.int32)
        t0 = time.perf_counter()
        if threads > 1:
            OD.batch_verify_parallel(pool, bits, sh.logit_dtype, truth[r].draft, n, np.zeros(B, np.int32),
                                     np.ones(B, np.uint8))
        else:
            OV.batch_verify(bits, sh.logit_dtype, truth[r].draft, n, np.zeros(B, np.int32), np.ones(B, np.uint8))
        t_ver.append(time.perf_counter() - t0)
    # KV copy rate of the oracle's gather: one whole 300-token member, every plane, into a
    # right-aligned staging row (per plane on its own thread when threads > 1)
    P, cap = sh.n_planes, 320
    src = W.gen_kv_bits_np(args.seed, 1 * P * sh.H * cap * sh.D).reshape(1, P, sh.H, cap, sh.D)
    dst = np.zeros((1, P, sh.H, cap, sh.D), np.uint16)

    def gather_plane(p):
        OA.copy_rows(src[:, p:p + 1], dst[:, p:p + 1], count=np.array([299]), src_row=np.array([0]),
                     dst_col=np.array([1]))
    t0 = time.perf_counter()
    if threads > 1:
        list(pool.map(gather_plane, range(P)))
    else:
        OA.copy_rows(src, dst, count=np.array([299]), src_row=np.array([0]), dst_col=np.array([1]))
    t_cp = time.perf_counter() - t0
    pool.shutdown()
    kv_rate = 2 * 299 * P * sh.H * sh.D * 2 / max(t_cp, 1e-9)   # bytes read + written per s
    t_total = t_plan + n_batches * float(np.mean(t_ver)) + kv_bytes / kv_rate
    parts = {"plan_s": t_plan, "verify_s_per_batch": float(np.mean(t_ver)), "batches": n_batches,
             "same_length_batches": n_same, "same_length_members": same_members,
             "fallback_members": fb_members, "kv_bytes": kv_bytes, "kv_copy_GBps": kv_rate / 1e9, "total_s": t_total, "threads": threads}
    return N / t_total, parts


def pool_sample_text(args, parts, threads):
    return (f"the oracle's GetBatch plan over the whole {args.pool_n}-sequence drain ({parts['batches']} "
            f"batches, timed in full); per-batch oracle verify timed on 2 batches and the KV gather of one "
            f"whole member (all 72 planes), extrapolated to the drain's batches and "
            f"{parts['kv_bytes'] / 1e9:.0f} GB; numpy, "
            + (f"thread-parallel driver on {threads} threads" if threads > 1 else "single thread")
            + f", on {cpu_info()}")


SLEEP_CYCLES = 200_000     # ~0.1 ms at 1.965 GHz: longer than Python's enqueue of one batch
ALG3_CHUNK = 64            # Alg. 3 device-loop iterations between host checks of the drain


def run_pool(args, rank, world, device, emulate=False):
    """EXSpec pool (BASELINE.json configs[4]): N Qwen3-shaped sequences, band-sharded over
    the ranks; each rank drains its shard (K4 plan, per batch gather / verify / write-back
    / scatter); one NCCL all-gather of outputs + counters at the end.  value = sequences/s
    over the whole job (max over ranks); strong scaling (N fixed)."""
    import torch
    import torch.distributed as dist

    from paper_2510_22876_b200 import _abi
    from paper_2510_22876_b200.dist import gather_results, shard_balanced, shard_bands, shard_strided
    from paper_2510_22876_b200.exspec import SequencePool

    sh = W.SHAPES["qwen3"]
    k, V, B = sh.k, sh.V, sh.B
    N = args.pool_n
    lens, order = pool_workload(args)
    if args.shard == "balanced":
        shards = shard_balanced(order, world, np.asarray(lens, np.float64) + args.shard_c * args.max_new)
    else:
        shards = (shard_bands if args.shard == "band" else shard_strided)(order, world)
    mine = shards[rank]
    n_loc = len(mine)
    cap = ((int(lens.max()) + args.max_new + k + 1) + 15) // 16 * 16
    Wn = min(args.pool_W or n_loc, 2048, n_loc)
    sp = SequencePool(n_loc, cap, sh.layers, sh.H, sh.D, k, W=Wn, B=min(B, Wn),
                      min_group=args.min_group, max_new=args.max_new, device=device, kv_init=False,
                      consumer=args.pool_consumer, verify_group=args.pool_verify_group,
                      scatter_stream=bool(args.pool_scatter_stream), patience=args.pool_patience,
                      pipeline=bool(args.pool_pipeline) and args.pool_mode == "epoch" and args.pool_exec == "native",
                      n_staging=args.pool_staging if args.pool_exec == "native" else 1)
    local_lens = lens[mine]
    local_order = np.arange(n_loc)            # `mine` is already in admission order
    ring_lg = [W.gen_logits_torch(args.seed, r, sp.B, k, V, sh.logit_dtype, device) for r in range(RING)]
    ring_dr = [torch.from_numpy(W.gen_round_truth(args.seed, r, sp.B, k, V, args.pattern, alpha=args.alpha).draft).to(device)
               for r in range(RING)]
    ctr = {"i": 0}

    def inputs(b):
        j = ctr["i"] % RING
        ctr["i"] += 1
        return ring_lg[j], ring_dr[j]

    ran = np.zeros(8, np.int64)
    alg3_iters = {"n": 0}     # device-loop iterations issued (Alg. 3 mode, native)

    if args.pool_exec == "native":
        sp.native(list(zip(ring_lg, ring_dr)), V=V, logit_dtype=ring_lg[0].dtype,
                  est_gather_GBps=args.pool_est[0], est_verify_us=args.pool_est[1])

    def drain(events=None, admit=None):
        # every drain is the same workload: the pool state and the input ring restart.
        # admit(): the e2e drain's own admission from pinned host buffers instead
        if admit is None:
            sp.load(local_lens, order=local_order)
        else:
            admit()
        ctr["i"] = 0
        sp.moved.zero_()
        epochs = batches = 0
        ran[:] = 0
        if args.pool_exec == "native" and events is None and args.pool_mode == "alg3":
            # Alg. 3 as printed on the device: chunks of plan -> batch 0 -> re-plan iterations
            # with no host sync inside a chunk (specdec_pool_alg3); drained-pool iterations
            # at the end of the last chunk are no-ops
            sp.alg3_exec.zero_() if getattr(sp, "alg3_exec", None) is not None else None
            alg3_iters["n"] = 0
            if args.alg3_graph and getattr(sp, "_alg3_gexec", None) is None:
                sp.alg3_native(RING)     # the first drain: direct launches set the kernels' attributes
                alg3_iters["n"] += RING
            while sp.has_active():
                if args.alg3_graph:      # a CUDA graph of RING iterations, replayed
                    sp.alg3_graph(ALG3_CHUNK // RING, conditional=args.alg3_graph == 2)
                else:
                    sp.alg3_native(ALG3_CHUNK)
                alg3_iters["n"] += ALG3_CHUNK
            ex = sp.alg3_exec.cpu().numpy()
            ran[0], ran[1], ran[2], ran[3] = ex[0], ex[1], ex[2], ex[3]
            return int(ex[0]), int(ex[0])
        if args.pool_exec == "native" and events is None:
            # the per-batch launch loop in C++ (csrc/pool_exec.cu), which counts its launches
            sp._launches.value = 0
            while True:
                r_run, r_same, m_same, m_fb = sp.epoch_native(1 if args.pool_mode == "alg3" else 0)
                if r_run == 0:
                    break
                epochs += 1
                batches += r_run
                ran[0] += r_run
                ran[1] += r_same
                ran[2] += m_same
                ran[3] += m_fb
            return epochs, batches
        while True:
            nb, kinds, blens, sizes = sp.plan()
            if nb == 0:
                break
            epochs += 1
            if args.pool_mode == "alg3":   # Alg. 3 as printed: batch 0, then re-plan
                nb = 1
            for b in range(nb):
                # counters of the batches that RAN: batches, same-length, their members,
                # fallback members (K4's own counters count planned batches)
                ran[0] += 1
                ran[1 if kinds[b] else 3] += 1 if kinds[b] else int(sizes[b])
                ran[2] += int(sizes[b]) if kinds[b] else 0
                lg, d = inputs(b)
                if events is not None:
                    fb = sp.moves_kv(kinds[b])
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    # keep the GPU busy while Python enqueues this batch, so that the event
                    # intervals hold kernel time only, not host launch gaps
                    torch.cuda._sleep(SLEEP_CYCLES)
                    e[0].record()
                    if fb:
                        sp.gather(b)
                    e[1].record()
                    sp.verify_writeback(b, lg, d, V)
                    e[2].record()
                    if fb:
                        sp.scatter(b, blens[b])
                    e[3].record()
                    events.append((fb, e))
                else:
                    sp.run_batch(b, kinds[b], blens[b], lg, d, V=V)
                batches += 1
        return epochs, batches

    drain()                                   # warm-up drain (attributes, allocator)
    if world > 1 and not emulate:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(device.index if device.index is not None else 0)
    reps = []
    with clocks:
        for _ in range(max(1, args.reps)):       # --reps R: median of R timed drains
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            if world > 1 and not emulate:
                dist.barrier()
            torch.cuda.synchronize()
            t0.record()
            epochs, batches = drain()
            # the only collective: finished outputs + counters, once, at the end
            counters = sp.counters.clone()
            t1.record()
            torch.cuda.synchronize()
            reps.append(t0.elapsed_time(t1))
    ms = float(np.median(reps))
    moved = int(sp.moved.item())
    cnt = ran.copy()          # executed batches (see drain); K4's counters: planned ones
    cnt[5] = int(counters[0].item())
    status = int(sp.status.item())
    out_loc = sp.out_buf.cpu().numpy()
    gen_loc = sp.gen.cpu().numpy()
    if emulate:
        # one rank's shard drained alone on this GPU (no collectives): see run_pool_emulated.
        # A second, serial drain with events around every launch splits the shard's time
        # into its two streams (fallback KV moves, verifies)
        assert int((gen_loc == args.max_new).sum()) == n_loc, "every sequence reaches max_new (EOS off)"
        evs = []
        drain(evs)
        torch.cuda.synchronize()
        return {"rank": rank, "ms": ms, "seqs": n_loc, "epochs": epochs, "batches": int(cnt[0]),
                "same_length_batches": int(cnt[1]), "fallback_batches": int(cnt[0]) - int(cnt[1]),
                "same_length_members": int(cnt[2]), "fallback_members": int(cnt[3]), "kv_bytes": moved,
                "status": status, "window": Wn,
                "prompt_len_range": [int(local_lens.min()), int(local_lens.max())],
                "prompt_tokens": int(local_lens.sum()), "clocks": clocks.summary(),
                "serial_ms": {"K2_gather_scatter": sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3])
                                                       for fb, e in evs if fb),
                              "K1_same_length": sum(e[1].elapsed_time(e[2]) for fb, e in evs if not fb),
                              "K1_fallback": sum(e[1].elapsed_time(e[2]) for fb, e in evs if fb)}}
    if world > 1:
        ms = max_over_ranks(ms, device, world)
        g0 = time.perf_counter()
        _, gen_all, cnt_all = gather_results(mine, out_loc, gen_loc, cnt, N, args.max_new,
                                             device=coll_device(device))
        gather_ms = (time.perf_counter() - g0) * 1e3
    else:
        gen_all, cnt_all, gather_ms = gen_loc, cnt, 0.0
    assert int((gen_all == args.max_new).sum()) == N, "every sequence reaches max_new (EOS off)"
    # e2e: the same drain through the public API with its host I/O inside the timed region --
    # the sequences admitted from pinned host buffers (prompt lengths, admission order,
    # prompt tokens [N, cap_tok]) and every generated token read back (out_buf, gen); the
    # per-batch logits are the model's, produced on the device (the executor's forward)
    e2e = None
    if not args.no_e2e:
        g = torch.Generator().manual_seed(args.seed)
        h_len = torch.as_tensor(local_lens, dtype=torch.int32).pin_memory()
        h_ord = torch.as_tensor(local_order, dtype=torch.int32).pin_memory()
        h_tok = torch.randint(2, V, (n_loc, sp.tokens.shape[1]), generator=g, dtype=torch.int64)
        h_tok[torch.arange(sp.tokens.shape[1])[None, :] >= torch.as_tensor(local_lens)[:, None]] = 0
        h_tok = h_tok.pin_memory()
        h_out = torch.empty(sp.out_buf.shape, dtype=sp.out_buf.dtype).pin_memory()
        h_gen = torch.empty(sp.gen.shape, dtype=sp.gen.dtype).pin_memory()

        def admit():
            sp.len.copy_(h_len, non_blocking=True)
            sp.order.copy_(h_ord, non_blocking=True)
            sp.tokens.copy_(h_tok, non_blocking=True)
            sp.gen.zero_()
            sp.active.fill_(1)
            sp.counters.zero_()
            sp.verify_calls = 0
            if getattr(sp, "_ring_pos", None) is not None:
                sp._ring_pos.value = 0
        ms_e = []
        for _ in range(max(1, args.reps)):
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0.record()
            drain(admit=admit)
            h_out.copy_(sp.out_buf, non_blocking=True)
            h_gen.copy_(sp.gen, non_blocking=True)
            t1.record()
            torch.cuda.synchronize()
            ms_e.append(t0.elapsed_time(t1))
        assert int((h_gen == args.max_new).sum()) == n_loc, "e2e: every sequence reaches max_new"
        bi = h_len.numel() * 4 + h_ord.numel() * 4 + h_tok.numel() * 8
        bo = h_out.numel() * 8 + h_gen.numel() * 4
        e2e_ms = max_over_ranks(float(np.median(ms_e)), device, world) if world > 1 else float(np.median(ms_e))
        e2e = {"value": N / (e2e_ms / 1e3), "unit": "sequences/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo,
               "note": "one drain per step: prompt lengths, order and tokens copied in from pinned host memory, "
                       "the generated tokens of every sequence read back, inside the timed region"}
    # second drain with events around the fallback batches' KV moves (roofline of K2)
    evs = []
    if rank == 0:
        drain(evs)
        torch.cuda.synchronize()
    k2_ms = sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for fb, e in evs if fb)
    k1_same_ms = sum(e[1].elapsed_time(e[2]) for fb, e in evs if not fb)
    k1_fb_ms = sum(e[1].elapsed_time(e[2]) for fb, e in evs if fb)
    moved2 = int(sp.moved.item()) if rank == 0 else 0
    peak, peak_src = peaks()
    achieved = moved2 / (k2_ms / 1e3) / 1e9 if k2_ms else 0.0
    rate_same = cnt_all[1] / max(1, cnt_all[0])
    roof = {"bound": "hbm", "kernel": "specdec_realign_kv gather+scatter (fallback batches)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
            # launches differ in size (one per fallback batch): no single per-launch
            # figure; the note gives the ncu traffic of one representative gather
            "traffic_note": ncu_traffic("pool_gather")[1], "peak_source": peak_src}
    if sp.consumer == "slot":
        # no KV moves: the dominant kernel is the verify (logits of every member row)
        lg_bytes = (int(cnt[2]) + int(cnt[3])) * (k + 1) * V * 2
        k1_ms = k1_same_ms + k1_fb_ms
        ach = lg_bytes / (k1_ms / 1e3) / 1e9 if k1_ms else 0.0
        roof = {"bound": "hbm", "kernel": "specdec_pool_verify (K1 + write-back), every batch",
                "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
                "note": "latency-bound launches of mean batch size "
                        f"{(int(cnt[2]) + int(cnt[3])) / max(1, int(cnt[0])):.2f}; event-timed one by one",
                "peak_source": peak_src}
    # the whole timed drain against the same peak: every algorithmic byte of the path -- the
    # KV moved by the gathers and scatters plus the logits every verified row reads ((k+1)
    # x V x 2 B) -- over the drain time.  With deferred fallback and 64-batch grouped
    # verifies the two kernels are about even (ncu launch list: K1 49 %, K2 45 %), so this is
    # the pool's own roofline; `roofline` keeps the K2 gather / scatter launches alone.
    lg_all = (int(cnt[2]) + int(cnt[3])) * (k + 1) * V * 2
    drain_gbps = (moved + lg_all) / (ms / 1e3) / 1e9 if ms else 0.0
    roof["drain"] = {"bytes": moved + lg_all, "kv_bytes": moved, "logit_bytes": lg_all,
                     "achieved": drain_gbps, "frac": drain_gbps / peak, "unit": "GB/s"}
    cb = pool_cpu_baseline(args) if (world == 1 and rank == 0) else None
    check = None
    if cb is not None:
        # the oracle's plan-driven drain (the cpu_baseline's own simulation) against the
        # counters of the timed GPU drain: the whole drain, not a sample
        o = cb["parts"]
        ours = {"batches": int(cnt_all[0]), "same_length_batches": int(cnt_all[1]),
                "same_length_members": int(cnt_all[2]), "fallback_members": int(cnt_all[3]),
                "kv_bytes": moved}
        ref = {key: int(o[key]) for key in ours}
        check = {"match": ours == ref, "ours": ours, "oracle": ref}
    return {
        "metric": "EXSpec pool sequences/s (Qwen3-8B shape, N=%d, B=%d, k=%d)" % (N, sp.B, k),
        "value": N / (ms / 1e3), "unit": "sequences/s", "n_gpus": world, "steps": epochs,
        "warmup": 1, "ms_per_step": ms / max(1, epochs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": sh.kv_dtype, "data": "synthetic",
        "config": {"workload": f"EXSpec pool drain: {N} seqs, prompt {args.pool_lengths} "
                               f"{'U[64,512]' if args.pool_lengths == 'random' else '256'}, max_new "
                               f"{args.max_new}, W={Wn}/rank, B={sp.B}, min_group={args.min_group}, "
                               f"sort on, {args.shard} shards, EOS off, mode {args.pool_mode}"
                               + (f" (deferred fallback, patience {args.pool_patience})"
                                  if args.pool_patience > 0 and args.pool_mode == "epoch" else "")
                               + (" (pipelined fallback: mixed batches beside the next plan)"
                                  if sp.pipeline else "")
                               + f", {args.pool_consumer} consumer, "
                               f"{args.pool_exec} launch loop"
                               + (f", fallback gathers overlapped ({sp.n_staging} staging buffers"
                                  + (", scatters on a third stream" if sp.scatter_stream else "") + ")"
                                  if args.pool_exec == "native" and sp.n_staging >= 2 else "")
                               + (f", up to {sp.verify_group} same-length batches per verify launch"
                                  if args.pool_exec == "native" and args.pool_mode == "epoch" and sp.verify_group > 1
                                  else "")
                               + (", Alg. 3 device loop replayed from a CUDA graph of 16 iterations"
                                  + (" with the KV moves in conditional nodes" if args.alg3_graph == 2 else "")
                                  if args.pool_exec == "native" and args.pool_mode == "alg3" and args.alg3_graph
                                  else ""),
                   "cap": cap, "pool_kv_GB_per_rank": sp.kv.numel() * 2 / 1e9,
                   "parallelism": f"pool sharded x{world}", "step": "one epoch (K4 plan + its batches)"},
        "pool": {"epochs": epochs, "batch_verifications": int(cnt_all[0]),
                 "grouping_rate": rate_same, "same_length_batches": int(cnt_all[1]),
                 "fallback_members": int(cnt_all[3]), "planned_batches_K4": int(cnt_all[5]),
                 "patience": args.pool_patience if args.pool_mode == "epoch" else 0,
                 "deferred_member_epochs": int(counters[7].item()),
                 "mean_batch": (int(cnt_all[2]) + int(cnt_all[3])) / max(1, int(cnt_all[0])),
                 "kv_bytes_moved_rank0": moved, "gather_ms": gather_ms,
                 "reps_drain_ms": reps if len(reps) > 1 else None,
                 # kernel time sums from a serial drain with events around every launch
                 # (rank 0): the overlapped executor's lower bound is max(K2, K1 same-length)
                 "serial_kernel_ms": {"K2_gather_scatter": k2_ms, "K1_same_length": k1_same_ms,
                                      "K1_fallback": k1_fb_ms, "drain_ms": ms}},
        "roofline": roof,
        "clocks": clocks.summary(), "status": status,
        # libspecdec launches in the timed drain: K4 per plan (the epochs + the final empty
        # plan), K1 with the fused write-back per batch, gather + scatter per fallback batch
        # (Alg. 3 device loop: K4 + gate + gather + verify + scatter per issued iteration)
        "gpu_launches": alg3_launches(sp, args, alg3_iters["n"], cnt) if alg3_iters["n"]
        else int(sp._launches.value) if args.pool_exec == "native" else (epochs + 1)
        + (_abi.specdec_verify_kernels(True) if sp.fused else _abi.specdec_verify_kernels(False) + 1) * int(cnt[0])
        + 2 * (int(cnt[0]) if sp.dense_consumer else 0 if sp.consumer == "slot" else int(cnt[0]) - int(cnt[1])),
        "e2e": e2e,
        "cpu_baseline": cb,
        "oracle_drain_check": check,
    }


def alg3_launches(sp, args, iters, cnt):
    """libspecdec kernels of the timed Alg. 3 drain: GetBatch + verify per iteration; the
    gather and scatter per iteration when launched as gated no-ops (direct loop), only for
    the batches that move KV in the graph's conditional nodes (none with the slot consumer)."""
    from paper_2510_22876_b200 import _abi
    kv1 = _abi.specdec_verify_kernels(True)
    if sp.consumer == "slot" and not os.environ.get("SPECDEC_ALG3_NOOP"):
        return (1 + kv1) * iters
    if args.alg3_graph != 2:
        return (3 + kv1) * iters
    moving = int(cnt[0]) if sp.consumer == "dense" else int(cnt[0]) - int(cnt[1])
    return (1 + kv1) * iters + 2 * moving


def pool_cpu_baseline(args):
    """The oracle on the same pool workload (bounded sample, a few seconds; see
    oracle_pool_sample), for the pool line's cpu_baseline."""
    if args.no_cpu_baseline:
        return None
    from oracle import driver as OD
    nthr = OD.host_threads()
    sps, parts = oracle_pool_sample(args, threads=nthr)
    sps1, parts1 = oracle_pool_sample(args, threads=1)
    return {"value": sps, "unit": "sequences/s", "cores": nthr, "kind": "oracle",
            "sample": pool_sample_text(args, parts, nthr), "nproc": nthr, "cpu_model": cpu_info(),
            "parts": parts, "single_thread": {"value": sps1, "cores": 1, "parts": parts1}}


def run_pool_emulated(args, device):
    """--emulate-ranks G on one GPU: drain each of the G band shards alone, one after the
    other, exactly as rank r of a G-GPU run would (same shard, same executor, no
    collective inside the drain).  The G-GPU job time is the slowest shard (the ranks
    share nothing until the end-of-run all-gather of ~2 MB), so the predicted whole-job
    throughput is N / max_r(ms_r).  This is a prediction from measured per-shard times,
    not a multi-GPU measurement."""
    import torch
    G = args.emulate_ranks
    per = []
    for r in range(G):
        per.append(run_pool(args, r, G, device, emulate=True))
        torch.cuda.empty_cache()
    mx = max(p["ms"] for p in per)
    N = args.pool_n
    return {
        "metric": "EXSpec pool sequences/s (Qwen3-8B shape, N=%d, B=8, k=5)" % N,
        "value": N / (mx / 1e3), "unit": "sequences/s", "n_gpus": 1, "steps": sum(p["epochs"] for p in per),
        "warmup": 1, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"EXSpec pool drain: {N} seqs, prompt {args.pool_lengths}, {args.shard} shards",
                   "parallelism": f"pool sharded x{G}, EMULATED: each shard drained alone on one B200"},
        "emulated": {"ranks": G, "predicted_seq_per_s": N / (mx / 1e3),
                     "per_rank_ms": [p["ms"] for p in per], "per_rank_seqs": [p["seqs"] for p in per],
                     "per_rank_batches": [p["batches"] for p in per],
                     "per_rank_kv_GB": [p["kv_bytes"] / 1e9 for p in per],
                     "per_rank_fallback_batches": [p["fallback_batches"] for p in per],
                     "per_rank_fallback_members": [p["fallback_members"] for p in per],
                     "per_rank_same_length_batches": [p["same_length_batches"] for p in per],
                     "per_rank_prompt_len_range": [p["prompt_len_range"] for p in per],
                     "per_rank_window": [p["window"] for p in per],
                     "per_rank_same_length_members": [p["same_length_members"] for p in per],
                     "per_rank_serial_ms": [p["serial_ms"] for p in per],
                     "total_kv_GB": sum(p["kv_bytes"] for p in per) / 1e9,
                     "total_batches": sum(p["batches"] for p in per),
                     "imbalance_max_over_mean": mx / (sum(p["ms"] for p in per) / G),
                     "note": "prediction: job time = slowest shard; the end-of-run all-gather (~2 MB over "
                             "NVLink) is not included"},
        "clocks": per[0]["clocks"], "status": max(p["status"] for p in per), "e2e": None, "cpu_baseline": None,
    }


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, rank 0 only."""
    if rank != 0:
        return None
    from oracle import driver as OD
    nthr = OD.host_threads()
    if args.config == "pool":
        t0 = time.perf_counter()
        sps, parts = oracle_pool_sample(args, threads=nthr)
        wall = time.perf_counter() - t0
        sample = pool_sample_text(args, parts, nthr)
        return {"impl": "reference", "metric": "EXSpec pool sequences/s (Qwen3-8B shape, N=%d, B=8, k=5)"
                % args.pool_n, "value": sps, "unit": "sequences/s", "n_gpus": world, "steps": 1,
                "warmup": 0, "ms_per_step": parts["total_s"] * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": f"EXSpec pool drain: {args.pool_n} seqs, prompt {args.pool_lengths}"},
                "cpu_baseline": {"value": sps, "unit": "sequences/s", "cores": nthr, "kind": "oracle",
                                 "sample": sample, "nproc": nthr, "cpu_model": cpu_info(), "parts": parts,
                                 "wall_s": wall},
                "e2e": {"value": sps, "unit": "sequences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    sh = shape_for(args)
    n = max(2, min(args.steps, 3))
    t0 = time.perf_counter()
    rps, parts = oracle_round_sample(sh, args, rounds=n, threads=nthr)
    wall = time.perf_counter() - t0
    sample = (f"{n} whole oracle rounds of the {sh.name} workload (verify over the full logits tail, repad, "
              f"realign over all {sh.n_planes} KV planes; no extrapolation), thread-parallel driver on {nthr} "
              f"threads (oracle/driver.py); numpy on {cpu_info()}")
    return {"impl": "reference", "metric": METRIC, "value": rps, "unit": "rounds/s",
            "n_gpus": world, "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 / rps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": sh.kv_dtype,
            "data": "synthetic", "config": {"workload": workload_name(sh, args)},
            "cpu_baseline": {"value": rps, "unit": "rounds/s", "cores": nthr, "kind": "oracle",
                             "sample": sample, "nproc": nthr, "cpu_model": cpu_info(), "parts_s": parts,
                             "wall_s": wall},
            "e2e": {"value": rps, "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out))
        return
    import torch
    import torch.distributed as dist
    # SPECDEC_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 over gloo, so the
    # N > 1 code path can be exercised on a one-GPU box; the real launch uses NCCL.
    shared = os.environ.get("SPECDEC_BENCH_SHARE_GPU") == "1"
    if shared:
        local = 0
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if args.config == "pool" and args.emulate_ranks > 1 and world == 1:
        print(json.dumps(run_pool_emulated(args, device)))
        return
    if args.config == "pool":
        out = run_pool(args, rank, world, device)
        if rank == 0:
            print(json.dumps(out))
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    res = run_ours(args, rank, world, device)
    sh = res["sh"]
    if rank == 0:
        peak, peak_src = peaks()
        value = world * args.steps / (res["ms"] / 1e3)
        k2_launch_ms = res["k2_ms"] / args.steps
        bytes_per_launch = res["moved"] / args.steps
        # (B=1 moves no KV: K2 is not launched and the roofline line reports 0 bytes)
        achieved = bytes_per_launch / (k2_launch_ms / 1e3) / 1e9 if k2_launch_ms > 1e-6 else 0.0
        traffic, traffic_note = ncu_traffic(f"{sh.name}_B{sh.B}" + (f"_ctx{args.ctx}" if args.ctx else "")
                                            + ("_pingpong" if args.kv_mode == "pingpong" else ""))
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = round_cpu_baseline(sh, args, rounds=2)
        out = {
            "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": sh.kv_dtype, "data": "synthetic",
            "config": {"workload": workload_name(sh, args), "B": sh.B, "k": sh.k, "V": sh.V,
                       "kv": f"{sh.layers}x{sh.H}x{sh.D} {sh.kv_dtype}", "cap": W.derive_cap(sh, args.warmup + args.steps + 2),
                       "width_end": res["end_width"],
                       "episode": (f"initial lengths restored every {args.episode} rounds by 3 device "
                                   f"copies inside the timed region (stationary workload)")
                       if args.episode else "none (contexts grow through the timed region)",
                       "l2": f"inputs > L2: {RING}-buffer logits ring ({RING * res['logits_bytes'] / 1e6:.0f} MB) "
                             f"and the KV cache (GB-scale); no flush needed",
                       "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm", "kernel": "specdec_realign_kv (K2)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_note": traffic_note, "peak_source": peak_src,
                         "bytes_per_launch": bytes_per_launch, "launch_ms": k2_launch_ms,
                         "kv_mode": args.kv_mode,
                         "copied_GBps": res["copied"] / args.steps / (k2_launch_ms / 1e3) / 1e9
                         if k2_launch_ms > 1e-6 else 0.0},
            "kernels_ms_per_step": {"verify_K1": res["k1_ms"] / args.steps,
                                    "repad_K3": res["k3_ms"] / args.steps,
                                    "realign_K2": k2_launch_ms},
            "verify_logits_GBps": res["logits_bytes"] / (res["k1_ms"] / args.steps / 1e3) / 1e9,
            # the whole round against the same peak: algorithmic bytes of K1 (logits) + K2
            # (region A's device counter: shifting rows only, in place) + K3 (tokens, masks,
            # positions at the mean width) per value-region round time
            "round_bandwidth": round_bandwidth(res, sh, args, peak),
            "clocks": res["clocks"],
            "e2e": res["e2e"],
            "gpu_launches": res["kernels_per_round"] * args.steps,
            "launch_mode": args.round_mode + (f" (one CUDA graph per {args.episode}-round episode: the "
                                              f"episode's state reset + its rounds; the rounds after the last "
                                              f"whole episode from a block graph of their own)"
                                              if args.round_mode == "graph-block" else
                                              " (graph: one CUDA graph per (parity, ring slot), 3 kernels per replay)"),
            "bytes_moved_check": {"value_region": res["moved_A"], "kernel_region": res["copied"]},
            "k2_per_launch": k2_spread(*res["k2_launches"], peak),
            # share of the kept KV bytes that K2 had to move (rows with a shift; f3 moves the
            # physical origin to shrink it), over the kernel-timing region's rounds
            "moved_share": {"value": res["moved"] / res["kept_bytes"] if res["kept_bytes"] else 0.0,
                            "moved_bytes": res["moved"], "all_kept_bytes": res["kept_bytes"],
                            "episode": args.episode},
            "reps": {"n": len(res["reps_ms"]), "ms_per_step": [x / args.steps for x in res["reps_ms"]],
                     "value": "median"} if len(res["reps_ms"]) > 1 else None,
            "status": res["status"],
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
