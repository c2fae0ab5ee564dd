#!/usr/bin/env python
"""bench.py -- the WindowQuant hot path on B200 (driver contract).

One STEP = one pass of the whole hot path over one batch in the
paper's serving setting (T5: the search and quantization run once per
request batch, then 50 tokens are generated):
    wq_window_scores -> wq_assign_bits (all L layers) -> L x (wq_layer_layout +
    wq_reorder_quantize_pack) -> 50 x L x wq_decode_attention
(+ one NCCL all-gather of (m, l, o) partials and wq_merge_partials per decode call
under the N > 1 sequence split).  value = generated tokens / s = B * 50 / step time.

Default workload: C5, the 7B long-video config the north-star targets are quoted
on (256 frames x 196 = 50,176 visual tokens, B = 4, 28 layers, S = 32,
widths {2,4,8,16}).  Inputs are seeded synthetic tensors resident in HBM;
28 layers x ~108 MB packed images >> 126 MB L2, so every decode call reads HBM.

--impl reference times the CPU oracle (oracle/, plain C fp64) on a bounded sample
of the same workload (there is no reference implementation; BASELINE.json).
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

from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn tokens/s + achieved HBM GB/s vs peak; quantize-pack GB/s (1/2/4/8 B200)"
UNIT = "tokens/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------------------
# clocks sampled DURING the timed region
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# the CUDA path
# ------------------------------------------------------------------------------------------
class Workload:
    """All inputs of one batch of cfg resident on the device, plus the output and
    scratch buffers of the path.  Under a sequence split each rank quantizes and
    decodes its share of every width segment (wq_shard_slots)."""

    def __init__(self, cfg, device, rank=0, world=1, n_gen=None, merge="peer", heads=None):
        import torch
        from paper_2605_02262_b200 import synth, wq
        self.torch, self.wq = torch, wq
        self.cfg, self.dev, self.rank, self.world = cfg, device, rank, world
        m = cfg.model
        # P1 head sharding: this rank's kv heads [h0, h1) of every request (the inputs are
        # generated for the full model shape and sliced, so the data is the full job's)
        h0, h1 = heads if heads is not None else (0, m.H)
        if (h0, h1) != (0, m.H):
            grp = m.Hq // m.H
            m = replace(m, H=h1 - h0, Hq=(h1 - h0) * grp)
        self.heads = (h0, h1)
        self.m = m
        self.L = cfg.layers
        self.n_gen = cfg.n_gen if n_gen is None else n_gen
        B = cfg.B
        self.g = wq.geom(B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
        self.opts = wq.AssignOpts(cfg.budget, 1, 0)
        self.thr = wq.wq_thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
        self.sm_scale = 1.0 / math.sqrt(m.d)
        # inputs
        self.vis, self.txt = synth.embeddings(B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, device)
        self.K, self.V, self.kr, self.vr = [], [], [], []
        hs = slice(h0, h1)
        qs = slice(h0 * (m.Hq // m.H), h1 * (m.Hq // m.H))
        for l in range(self.L):
            K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, device)
            if (h0, h1) != (0, cfg.model.H):
                K, V, kr, vr = (x[:, hs].contiguous() for x in (K, V, kr, vr))
            self.K.append(K); self.V.append(V); self.kr.append(kr); self.vr.append(vr)
        base = int(rest_len[0].item())
        steps = [[base + t + 1] * B for t in range(self.n_gen)]
        self.rest_len = torch.tensor(steps, dtype=torch.int32, device=device)       # [n_gen][B]
        self.rest_zero = torch.zeros((B,), dtype=torch.int32, device=device)
        self.q = torch.stack([torch.stack([synth.queries(B, cfg.model.Hq, cfg.model.H, m.d, cfg.seed, l, t,
                                                         device)[:, qs].contiguous()
                                           for l in range(self.L)]) for t in range(self.n_gen)])
        # path buffers
        W = cfg.W
        self.scores = torch.empty((B, W), dtype=torch.float64, device=device)
        self.sws = torch.empty(wq.wq_window_scores_workspace(B, m.D), dtype=torch.uint8, device=device)
        self.bits = torch.empty((self.L, B, W), dtype=torch.uint8, device=device)
        self.rank_t = torch.empty((B, W), dtype=torch.int32, device=device)
        self.perm = torch.empty((self.L, B, W), dtype=torch.int32, device=device)
        self.seg = torch.empty((self.L, B, 5), dtype=torch.int32, device=device)
        self.perm_r = torch.empty((self.L, B, W), dtype=torch.int32, device=device)
        self.seg_r = torch.empty((self.L, B, 5), dtype=torch.int32, device=device)
        self.offs = torch.empty((self.L, B * m.H + 1), dtype=torch.int64, device=device)
        self.dws = torch.zeros(wq.wq_decode_workspace(self.g), dtype=torch.uint8, device=device)
        self.out = torch.empty((self.n_gen, self.L, B, m.Hq, m.d), dtype=torch.float16, device=device)
        self.part = torch.empty((B, m.Hq, m.d + 2), dtype=torch.float32, device=device) if world > 1 else None
        self.gathered = (torch.empty((world, B, m.Hq, m.d + 2), dtype=torch.float32, device=device)
                         if world > 1 else None)
        # cross-GPU merge of the sequence split: fused peer-memory exchange (default) or
        # partial -> NCCL all-gather -> wq_merge_partials (merge="nccl", the baseline)
        self.peer, self.merge_note = None, None
        if world > 1 and merge == "peer":
            try:
                from paper_2605_02262_b200.parallel import PeerMerge
                self.peer = PeerMerge(self.g, device=device)
            except Exception as e:                           # no IPC / peer access: NCCL path
                self.merge_note = f"peer setup failed ({type(e).__name__}: {e}); NCCL all-gather used"
        # size the packed images once (setup, untimed): they depend only on the inputs
        self.packed = None
        self._setup_pass()

    def _setup_pass(self):
        torch, wq = self.torch, self.wq
        self.search()
        for l in range(self.L):
            wq.wq_layer_layout(self.g, self.seg_r[l], self.offs[l])
        torch.cuda.synchronize()
        sizes = self.offs[:, -1].cpu().tolist()
        self.packed = [torch.zeros(int(s) + 16, dtype=torch.uint8, device=self.dev) for s in sizes]
        self.packed_bytes = [int(s) for s in sizes]
        seg = self.seg.cpu().numpy()
        self.class_windows = (seg[:, :, 1:] - seg[:, :, :-1]).sum(axis=(0, 1)).tolist()

    # --- the four calls ---
    def search(self):
        wq = self.wq
        wq.wq_window_scores(self.vis, self.txt, self.cfg.S, scores=self.scores, workspace=self.sws)
        wq.wq_assign_bits(self.scores, self.thr, self.L, self.g, self.opts, self.bits, self.rank_t, self.perm,
                          self.seg)
        if self.world > 1:
            for l in range(self.L):
                wq.wq_shard_slots(self.perm[l], self.seg[l], self.world, self.rank, self.perm_r[l], self.seg_r[l])
        else:
            self.perm_r, self.seg_r = self.perm, self.seg

    def quantize(self):
        wq = self.wq
        for l in range(self.L):
            wq.wq_layer_layout(self.g, self.seg_r[l], self.offs[l])
            wq.wq_reorder_quantize_pack(self.K[l], self.V[l], 0, self.g, self.perm_r[l], self.seg_r[l],
                                        self.offs[l], self.packed[l])

    def decode(self, group=None):
        torch, wq = self.torch, self.wq
        for t in range(self.n_gen):
            rl = self.rest_len[t] if self.rank == 0 else self.rest_zero
            for l in range(self.L):
                # every decode but the first after quantize follows work that does not
                # write the packed cache / offs / seg_off / rest_len: WQ_DECODE_EARLY
                # lets it plan and prefetch the cache while that work drains (PDL)
                flags = 0 if (t == 0 and l == 0) else wq.WQ_DECODE_EARLY
                if self.world == 1:
                    wq.wq_decode_attention(self.q[t, l], self.packed[l], self.offs[l], self.seg_r[l], self.g,
                                           self.kr[l], self.vr[l], rl, self.sm_scale, out=self.out[t, l],
                                           workspace=self.dws, flags=flags)
                elif self.peer is not None:
                    # fused path: the decode kernel exchanges the (m, l, o) partials over
                    # NVLink peer memory and merges them (no NCCL call, no merge kernel)
                    wq.wq_decode_attention_peer(self.q[t, l], self.packed[l], self.offs[l], self.seg_r[l], self.g,
                                                self.kr[l], self.vr[l], rl, self.sm_scale, self.out[t, l],
                                                self.peer.ptrs, self.peer.local, self.world, self.rank,
                                                self.peer.next_epoch(), workspace=self.dws)
                    if self.peer.epoch == 1 and not self._peer_checked(group):
                        continue                                 # fell back to NCCL (call redone there)
                else:
                    wq.wq_decode_attention(self.q[t, l], self.packed[l], self.offs[l], self.seg_r[l], self.g,
                                           self.kr[l], self.vr[l], rl, self.sm_scale, partial=self.part,
                                           workspace=self.dws, flags=flags)
                    self._all_gather(group)
                    wq.wq_merge_partials(self.gathered, self.g, out=self.out[t, l])

    def _all_gather(self, group):
        """partials of every rank into self.gathered: one NCCL all-gather (the gloo
        backend of the CPU-collective test runs takes the list form)."""
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(self.gathered, self.part, group=group)
        else:
            dist.all_gather(list(self.gathered.unbind(0)), self.part, group=group)

    def _peer_checked(self, group):
        """After the first fused call: every rank checks its timeout flag, and if any rank's
        wait timed out all ranks switch to the NCCL path (decided collectively) and redo
        the call that way.  Returns True if the fused path stays."""
        import torch
        import torch.distributed as dist
        bad = torch.tensor([1.0 if self.peer.timed_out() else 0.0], device=self.dev)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
        if bad.item() == 0.0:
            return True
        self.peer = None
        self.merge_note = "peer-memory exchange timed out at the first call; NCCL all-gather used"
        wq = self.wq
        rl = self.rest_len[0] if self.rank == 0 else self.rest_zero
        wq.wq_decode_attention(self.q[0, 0], self.packed[0], self.offs[0], self.seg_r[0], self.g, self.kr[0],
                               self.vr[0], rl, self.sm_scale, partial=self.part, workspace=self.dws)
        self._all_gather(group)
        wq.wq_merge_partials(self.gathered, self.g, out=self.out[0, 0])
        return False

    def launches_per_step(self):
        per_dec = 1 if (self.world == 1 or self.peer is not None) else 2
        shard = self.L if self.world > 1 else 0
        return 2 + 2 + shard + 2 * self.L + self.n_gen * self.L * per_dec

    def decode_bytes_per_call(self, l):
        """Algorithmic bytes of one wq_decode_attention launch: the
        packed image + FP16 rest tokens (K and V) + q read + out written."""
        cfg, m = self.cfg, self.m
        rest_tok = (cfg.tail + cfg.n_text + self.n_gen / 2 + 0.5) if self.rank == 0 else 0
        rest = cfg.B * m.H * rest_tok * m.d * 4
        qo = 2 * cfg.B * m.Hq * m.d * 2
        return self.packed_bytes[l] + rest + qo

    def quant_bytes_per_call(self, l):
        """read fp16 K+V of the rank's windows + write the packed image."""
        cfg, m = self.cfg, self.m
        n_win = int(self.seg_r[l][:, 4].sum().item())
        return n_win * m.H * cfg.S * m.d * 4 + self.packed_bytes[l]


def build_step(w, group, stream, use_graph: bool, warmup: int):
    """The timed step of bench.py (also driven by tests/test_gpu_fullsize.py so the
    parity check runs this exact launch path): search -> quantize -> decode, with
    `warmup` eager passes first; under use_graph the step's launches are captured in two
    CUDA graphs (search + quantize, decode) and replayed -- same kernels, same
    arguments, PDL-chained decodes (WQ_DECODE_EARLY) inside the decode graph.
    step(ev) records ev[0] / ev[1] around the decode phase."""
    import torch

    def step(ev=None):
        w.search()
        w.quantize()
        if ev is not None:
            ev[0].record(stream)
        w.decode(group)
        if ev is not None:
            ev[1].record(stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if not use_graph:
        return step
    g_sq, g_dec = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_sq):
        w.search()
        w.quantize()
    with torch.cuda.graph(g_dec):
        w.decode(group)
    torch.cuda.synchronize()
    w._graphs = (g_sq, g_dec)                               # keep the graphs alive with the workload

    def gstep(ev=None):
        g_sq.replay()
        if ev is not None:
            ev[0].record(stream)
        g_dec.replay()
        if ev is not None:
            ev[1].record(stream)

    gstep()
    torch.cuda.synchronize()
    return gstep


def _allreduce_max(t, group=None):
    """max over ranks of a small device tensor (NCCL), through the host for gloo."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t
    c = t.cpu()
    dist.all_reduce(c, op=dist.ReduceOp.MAX, group=group)
    return c.to(t.device)


def run_wq(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2605_02262_b200 import configs, wq
    local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wq.load(build_if_missing=False)
    cfg = configs.CONFIGS[args.config]
    if args.layers:
        cfg = cfg.with_(layers=args.layers)
    # multi-GPU mode: P2 sequence split (long video, C5) with the fused
    # cross-GPU merge, or P1 over (request, kv-head) units (C2-C4, or --parallel units):
    # rank r takes whole requests, or kv heads of one request when ranks outnumber
    # requests -- independent units, no collective on the data path
    mode = args.parallel if args.parallel != "auto" else ("seqsplit" if cfg.idx == 5 else "units")
    if world > 1 and mode in ("batch", "units"):
        from paper_2605_02262_b200.parallel import unit_shard
        b0, b1, h0, h1 = unit_shard(cfg.B, cfg.model.H, world, rank)
        cfg_global = cfg
        cfg = cfg.with_(B=b1 - b0)
        w = Workload(cfg, dev, 0, 1, n_gen=args.n_gen, heads=(h0, h1))
        mode = "batch" if (h0, h1) == (0, cfg.model.H) else "heads"
        w_world = 1
    else:
        cfg_global = cfg
        w = Workload(cfg, dev, rank, world, n_gen=args.n_gen, merge=args.merge)
        w_world = world
    group = dist.group.WORLD if world > 1 else None
    stream = torch.cuda.current_stream()
    use_graph = w_world == 1 and not args.no_graph
    step = build_step(w, group, stream, use_graph, args.warmup)
    if world > 1:
        dist.barrier()
    ev_all = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_dec = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        ev_all[0].record(stream)
        for s in range(args.steps):
            step(ev_dec[s])
            if w.peer is not None and w.peer.timed_out():          # fused merge: fail loudly, at once
                raise RuntimeError(f"fused cross-GPU merge: a peer wait timed out in step {s}")
        ev_all[1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if w.peer is not None and w.peer.timed_out():
        raise RuntimeError("fused cross-GPU merge: a peer wait timed out (outputs invalid)")
    total_ms = ev_all[0].elapsed_time(ev_all[1])
    dec_ms = sum(e[0].elapsed_time(e[1]) for e in ev_dec)
    # isolated wq_reorder_quantize_pack timing for the quantize GB/s figure: the L layers'
    # layouts first (untimed, they are separate wq_layer_layout calls), then one timed
    # pass of the L quantize launches back to back
    for l in range(w.L):
        w.wq.wq_layer_layout(w.g, w.seg_r[l], w.offs[l])
    qe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    qe[0].record(stream)
    for l in range(w.L):
        w.wq.wq_reorder_quantize_pack(w.K[l], w.V[l], 0, w.g, w.perm_r[l], w.seg_r[l], w.offs[l], w.packed[l])
    qe[1].record(stream)
    torch.cuda.synchronize()
    quant_ms = qe[0].elapsed_time(qe[1])
    t = torch.tensor([total_ms, dec_ms, quant_ms], dtype=torch.float64, device=dev)
    if world > 1:
        t = _allreduce_max(t)
    total_ms, dec_ms, quant_ms = t.tolist()

    ms_per_step = total_ms / args.steps
    tokens = cfg_global.B * w.n_gen                        # whole job: every rank's requests
    value = tokens / (ms_per_step / 1e3)
    n_dec = args.steps * w.n_gen * cfg.layers
    dec_launch_us = dec_ms * 1e3 / n_dec
    dec_bytes = float(np.mean([w.decode_bytes_per_call(l) for l in range(cfg.layers)]))
    peak, peak_src = peaks()
    achieved = dec_bytes / (dec_launch_us * 1e-6) / 1e9
    q_bytes = float(sum(w.quant_bytes_per_call(l) for l in range(cfg.layers)))
    q_gbs = q_bytes / (quant_ms * 1e-3) / 1e9
    # traffic: DRAM bytes of one decode launch from an `ncu --set full` capture of this
    # config (not measured in this run; the capture is named in traffic_source)
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "decode_dram_bytes.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get(cfg.name)
            traffic_src = tj.get("_source") if traffic is not None else None
        except Exception:
            traffic = None
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (seeded; shapes of LLaVA-OneVision-7B / Qwen2-7B video workloads)",
        "config": {"workload": cfg_global.name, "model_shape": cfg.model.name, "layers": cfg.layers,
                   "batch": cfg_global.B, "batch_per_gpu": cfg.B,
                   "visual_tokens": cfg.M, "window": cfg.S, "widths": list(cfg.widths), "gen_tokens": w.n_gen,
                   "parallelism": (f"{mode}{world}" if world > 1 else "single"),
                   "merge": (("fused peer-memory LSE merge" if w.peer is not None else (w.merge_note or
                              "NCCL all-gather + wq_merge_partials")) if w_world > 1 else None),
                   "launch": "cuda-graph replay" if use_graph else "host launches",
                   "l2": f"inputs > L2: {cfg.layers} layers x {w.packed_bytes[0] / 1e6:.0f} MB packed rotated",
                   "window_mix": dict(zip(["2", "4", "8", "16"], [int(x) for x in w.class_windows]))},
        "roofline": {"bound": "hbm", "kernel": "wq_decode_attention", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "bytes_per_launch": round(dec_bytes), "avg_launch_us": round(dec_launch_us, 3),
                     "peak_source": peak_src},
        "quantize": {"kernel": "wq_reorder_quantize_pack", "GB/s": round(q_gbs, 1),
                     "frac": round(q_gbs / peak, 4), "ms_per_L_layers": round(quant_ms, 3),
                     "bytes_L_layers": round(q_bytes)},
        "decode_only_tokens_per_s": round(cfg_global.B / (dec_launch_us * 1e-6 * cfg.layers), 1),
        "gpu_launches": w.launches_per_step() * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_ablation:
        result["ablation_unfused_t9"] = run_ablation_unfused(w, stream)
        result["ablation_unreordered_t8"] = run_ablation_unreordered(w, stream)
        result["ablation_similarity_t11"] = run_ablation_similarity(w, stream)
        result["ablation_group_quantizer"] = run_ablation_group(w, stream)
        result["ablation_search"] = run_ablation_search(w, stream)
    if not args.no_e2e:
        # every rank runs the end-to-end steps (the sequence split's decodes are
        # collective); the time is the max over ranks, the value the whole job's tokens
        e2e = run_e2e(w, args, stream, tokens=cfg_global.B * w.n_gen, group=group if world > 1 else None)
        if rank == 0:
            result["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(cfg, w, args)
    return result


def run_ablation_unfused(w, stream, n_layers=4, reps=5):
    """SURVEY §8(f) row 3 / the paper's fusion ablation (T9): per decode
    step the unfused path dequantizes the layer's cache to FP16 in HBM
    (wq_dequantize_image) and then runs FP16 attention over it; the fused path is
    wq_decode_attention on the packed image.  Per-layer device times over n_layers
    rotated layers (each image >> L2), reps passes each."""
    import torch
    wq = w.wq
    L = min(n_layers, w.L)
    imgs = []
    for l in range(L):
        seg16, offs16 = wq.wq_dequant_layout(w.g, w.seg_r[l])
        img16 = torch.zeros(int(offs16[-1].item()) + 16, dtype=torch.uint8, device=w.dev)
        imgs.append((seg16, offs16, img16))
    rl = w.rest_len[0]

    def fused(l):
        wq.wq_decode_attention(w.q[0, l], w.packed[l], w.offs[l], w.seg_r[l], w.g, w.kr[l], w.vr[l], rl,
                               w.sm_scale, out=w.out[0, l], workspace=w.dws)

    def dequant(l):
        seg16, offs16, img16 = imgs[l]
        wq.wq_dequantize_image(w.packed[l], w.offs[l], w.seg_r[l], w.g, offs16, img16)

    def dec16(l):
        seg16, offs16, img16 = imgs[l]
        wq.wq_decode_attention(w.q[0, l], img16, offs16, seg16, w.g, w.kr[l], w.vr[l], rl, w.sm_scale,
                               out=w.out[0, l], workspace=w.dws)

    def timed(fn):
        for l in range(L):
            fn(l)                                          # warm-up pass
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            for l in range(L):
                fn(l)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (reps * L)       # us per layer call

    t_f, t_d, t_16 = timed(fused), timed(dequant), timed(dec16)
    del imgs
    peak, _ = peaks()
    dq_bytes = float(w.packed_bytes[0] + imgs_bytes(w, 0))
    return {"fused_decode_us": round(t_f, 2), "dequantize_us": round(t_d, 2), "fp16_decode_us": round(t_16, 2),
            "dequantize_GBps": round(dq_bytes / (t_d * 1e-6) / 1e9, 1),
            "unfused_at_hbm_floor_us": round(dq_bytes / (peak * 1e9) * 1e6 + t_16, 2),
            "unfused_us": round(t_d + t_16, 2), "unfused_over_fused": round((t_d + t_16) / t_f, 3),
            "fp16_image_MB": round(imgs_bytes(w, 0) / 1e6, 1), "packed_image_MB": round(w.packed_bytes[0] / 1e6, 1),
            "paper": "T9 (P:1026-1027, A800): attention per layer per token 0.82 ms fused vs 1.25 ms unfused "
                     "(ratio 1.52)"}


def run_ablation_unreordered(w, stream, n_layers=4, reps=5):
    """SURVEY §8(f) row 1 / the paper's reordering ablation (T8, "Module III
    off"): the same records stored in original window order (wq_unreorder_image) and
    decoded in that order with a per-window width dispatch, against the reordered decode.
    Per-layer device times over n_layers rotated layers, reps passes each."""
    import torch
    wq = w.wq
    L = min(n_layers, w.L)
    ur = []
    for l in range(L):
        woff = wq.wq_unreordered_layout(w.g, w.bits[l].contiguous())
        uimg = torch.zeros_like(w.packed[l])
        wq.wq_unreorder_image(w.packed[l], w.offs[l], w.seg_r[l], w.perm_r[l], w.g, woff, uimg)
        ur.append((woff, uimg))
    rl = w.rest_len[0]

    def reordered(l):
        wq.wq_decode_attention(w.q[0, l], w.packed[l], w.offs[l], w.seg_r[l], w.g, w.kr[l], w.vr[l], rl,
                               w.sm_scale, out=w.out[0, l], workspace=w.dws)

    def unreordered(l):
        woff, uimg = ur[l]
        wq.wq_decode_attention_unreordered(w.q[0, l], uimg, w.offs[l], w.seg_r[l], woff, w.g, w.kr[l], w.vr[l],
                                           rl, w.sm_scale, out=w.out[0, l], workspace=w.dws)

    def timed(fn):
        for l in range(L):
            fn(l)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            for l in range(L):
                fn(l)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (reps * L)

    t_r, t_u = timed(reordered), timed(unreordered)
    del ur
    return {"reordered_decode_us": round(t_r, 2), "unreordered_decode_us": round(t_u, 2),
            "unreordered_over_reordered": round(t_u / t_r, 3),
            "paper": "T8 (P:1006-1008, A800, whole model): 1250 tokens/s with reordering vs 500 without (2.5x)"}


def run_ablation_similarity(w, stream, reps=5):
    """The paper's similarity-function comparison (T11): window scoring
    (wq_window_scores) with cosine (Eq.8) vs Pearson correlation on the bench workload."""
    import torch
    wq = w.wq
    out = {}
    for name, metric in (("cosine_us", wq.WQ_SIM_COSINE), ("pearson_us", wq.WQ_SIM_PEARSON)):
        wq.wq_window_scores(w.vis, w.txt, w.cfg.S, scores=w.scores, workspace=w.sws, metric=metric)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            wq.wq_window_scores(w.vis, w.txt, w.cfg.S, scores=w.scores, workspace=w.sws, metric=metric)
        e1.record(stream)
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) * 1e3 / reps, 1)
    out["visual_MB"] = round(w.vis.numel() * 2 / 1e6, 1)
    out["paper"] = ("T11 (P:1059-1061, batch 1, 100 frames): cosine 48 ms, Pearson 55 ms, Euclidean 49 ms; "
                    "cosine kept (Euclidean not provided here, include/wq.h)")
    return out


def _timed_layers(fn, L, stream, reps):
    """us per call of fn(l) over L rotated layers (one warm-up pass, reps timed passes)."""
    import torch
    for l in range(L):
        fn(l)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        for l in range(L):
            fn(l)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * L)


def run_ablation_group(w, stream, n_layers=4, reps=5):
    """the paper-literal group quantizer (WQ_GRAN_GROUP: one (s, mn) per
    (window, head, K|V), reading Q37) against the default per-channel K / per-token V
    parameters (Q19) on the bench workload: packed bytes, quantize and decode device time
    per layer call (n_layers rotated layers, reps passes)."""
    import torch
    wq = w.wq
    L = min(n_layers, w.L)
    GR = wq.WQ_GRAN_GROUP
    offs_g = [wq.wq_layer_layout(w.g, w.seg_r[l], gran=GR) for l in range(L)]
    torch.cuda.synchronize()
    bytes_g = [int(o[-1].item()) for o in offs_g]
    imgs_g = [torch.zeros(n + 16, dtype=torch.uint8, device=w.dev) for n in bytes_g]
    rl = w.rest_len[0]

    def quant(gran):
        def f(l):
            offs, img = (offs_g[l], imgs_g[l]) if gran else (w.offs[l], w.packed[l])
            wq.wq_reorder_quantize_pack(w.K[l], w.V[l], 0, w.g, w.perm_r[l], w.seg_r[l], offs, img, gran=gran)
        return f

    def dec(gran):
        def f(l):
            offs, img = (offs_g[l], imgs_g[l]) if gran else (w.offs[l], w.packed[l])
            wq.wq_decode_attention(w.q[0, l], img, offs, w.seg_r[l], w.g, w.kr[l], w.vr[l], rl, w.sm_scale,
                                   out=w.out[0, l], workspace=w.dws, flags=wq.WQ_DECODE_GROUP if gran else 0)
        return f

    tq0, tq1 = _timed_layers(quant(0), L, stream, reps), _timed_layers(quant(GR), L, stream, reps)
    td0, td1 = _timed_layers(dec(0), L, stream, reps), _timed_layers(dec(GR), L, stream, reps)
    b0 = sum(w.packed_bytes[:L]) / L
    b1 = sum(bytes_g) / L
    rest = w.decode_bytes_per_call(0) - w.packed_bytes[0]
    del imgs_g
    return {"packed_MB_per_layer": {"channel_token": round(b0 / 1e6, 2), "group": round(b1 / 1e6, 2)},
            "group_over_channel_token_bytes": round(b1 / b0, 4),
            "quantize_us": {"channel_token": round(tq0, 2), "group": round(tq1, 2)},
            "decode_us": {"channel_token": round(td0, 2), "group": round(td1, 2)},
            "decode_GBps": {"channel_token": round((b0 + rest) / (td0 * 1e-6) / 1e9, 1),
                            "group": round((b1 + rest) / (td1 * 1e-6) / 1e9, 1)},
            "note": "same windows, widths and kernels' structure; group = 16 B of parameters per record "
                    "instead of 4(d + S)"}


def run_ablation_search(w, stream, reps=5):
    """SURVEY §8(f) row 4 and the fused search: (a) the unfused chain wq_window_scores +
    wq_assign_bits (the bench step's search), (b) wq_search (one cooperative launch, the
    same results), (c) the per-layer K/Q scorer (wq_window_scores_layer: visual keys of
    layer l vs that layer's text queries, reading Q36) + a per-layer assignment -- L calls
    each.  Device time per search of all L layers."""
    import torch
    from paper_2605_02262_b200 import synth
    wq, cfg, m = w.wq, w.cfg, w.m
    L, B, W = w.L, cfg.B, cfg.W
    fo = (w.scores, w.bits, w.rank_t, w.perm, w.seg)
    qt = synth.text_queries(B, m.Hq, cfg.n_text, m.d, cfg.seed, 0, w.dev)
    sl = torch.empty((B, W), dtype=torch.float64, device=w.dev)
    lws = torch.empty(wq.wq_window_scores_workspace(B, m.H * m.d), dtype=torch.uint8, device=w.dev)
    bl = torch.empty((1, B, W), dtype=torch.uint8, device=w.dev)
    rk = torch.empty((B, W), dtype=torch.int32, device=w.dev)
    pl = torch.empty((1, B, W), dtype=torch.int32, device=w.dev)
    sg = torch.empty((1, B, 5), dtype=torch.int32, device=w.dev)

    def chain(_):
        w.search()

    def fused(_):
        wq.wq_search(w.vis, w.txt, w.thr, L, w.g, w.opts, outs=fo)

    def per_layer(_):
        for l in range(L):
            wq.wq_window_scores_layer(w.K[l], 0, qt, cfg.M, cfg.S, scores=sl, workspace=lws)
            wq.wq_assign_bits(sl, w.thr, 1, w.g, w.opts, bl, rk, pl, sg)

    t_c = _timed_layers(chain, 1, stream, reps)
    t_f = _timed_layers(fused, 1, stream, reps)
    t_l = _timed_layers(per_layer, 1, stream, reps)
    w.search()                                              # restore the step's plan
    torch.cuda.synchronize()
    return {"chain_us": round(t_c, 1), "fused_us": round(t_f, 1), "per_layer_scorer_us": round(t_l, 1),
            "fused_over_chain": round(t_f / t_c, 3),
            "layers": L, "note": "chain = the step's search; fused = wq_search (bit-identical outputs); "
                                 "per_layer = L x (wq_window_scores_layer + wq_assign_bits with L = 1)"}


def imgs_bytes(w, l):
    """bytes of layer l's FP16 image: every slot at 4*S*d bytes per (b, h)."""
    n_slots = int(w.seg_r[l][:, 4].sum().item())
    return n_slots * w.m.H * 4 * w.cfg.S * w.m.d


def run_e2e(w, args, stream, tokens=None, group=None):
    """Same metric through the public API with HOST inputs: every step copies its
    inputs (embeddings, per-layer K/V + rest, queries) from pinned host memory and
    reads all decode outputs back, inside the timed region.  The uploads run on a copy
    stream into two alternating device input sets, so step i+1's inputs cross PCIe while
    step i computes (a serving pipeline: the copy engine and the SMs work concurrently;
    step i's compute waits for its own upload, an upload waits until the compute that
    last used its set is done).  The timed region starts before the first upload and
    ends after the last step's outputs are back on the host."""
    import torch
    dev = w.dev
    host = {}
    for n in ("vis", "txt"):
        host[n] = getattr(w, n).cpu().pin_memory()
    hK = [k.cpu().pin_memory() for k in w.K]
    hV = [v.cpu().pin_memory() for v in w.V]
    hkr = [k.cpu().pin_memory() for k in w.kr]
    hvr = [v.cpu().pin_memory() for v in w.vr]
    hq = w.q.cpu().pin_memory()
    hout = torch.empty(w.out.shape, dtype=w.out.dtype).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in [host["vis"], host["txt"], hq] + hK + hV + hkr + hvr)
    d2h = hout.numel() * hout.element_size()
    steps = max(1, min(args.steps, 4))
    # two device input sets: the workload's own and a second one of the same shapes
    sets = [dict(vis=w.vis, txt=w.txt, K=w.K, V=w.V, kr=w.kr, vr=w.vr, q=w.q),
            dict(vis=torch.empty_like(w.vis), txt=torch.empty_like(w.txt), K=[torch.empty_like(x) for x in w.K],
                 V=[torch.empty_like(x) for x in w.V], kr=[torch.empty_like(x) for x in w.kr],
                 vr=[torch.empty_like(x) for x in w.vr], q=torch.empty_like(w.q))]
    cs = torch.cuda.Stream(device=dev)
    up = [torch.cuda.Event(), torch.cuda.Event()]
    free = [None, None]

    def upload(si):
        s = sets[si]
        with torch.cuda.stream(cs):
            if free[si] is not None:
                cs.wait_event(free[si])
            s["vis"].copy_(host["vis"], non_blocking=True)
            s["txt"].copy_(host["txt"], non_blocking=True)
            s["q"].copy_(hq, non_blocking=True)
            for l in range(w.L):
                s["K"][l].copy_(hK[l], non_blocking=True)
                s["V"][l].copy_(hV[l], non_blocking=True)
                s["kr"][l].copy_(hkr[l], non_blocking=True)
                s["vr"][l].copy_(hvr[l], non_blocking=True)
            up[si].record(cs)

    def compute(si):
        s = sets[si]
        stream.wait_event(up[si])
        w.vis, w.txt, w.K, w.V, w.kr, w.vr, w.q = s["vis"], s["txt"], s["K"], s["V"], s["kr"], s["vr"], s["q"]
        w.search()
        w.quantize()
        w.decode(group)
        hout.copy_(w.out, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        free[si] = ev

    def run(n, e_start=None):
        if e_start is not None:
            cs.wait_event(e_start)                 # the first upload is inside the timed region
        upload(0)
        for i in range(n):
            if i + 1 < n:
                upload((i + 1) % 2)
            compute(i % 2)

    import torch.distributed as dist
    run(2)                                         # warm-up (both sets)
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier(group=group)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(steps, e0)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # the workload keeps its own input set
    s0 = sets[0]
    w.vis, w.txt, w.K, w.V, w.kr, w.vr, w.q = s0["vis"], s0["txt"], s0["K"], s0["V"], s0["kr"], s0["vr"], s0["q"]
    del sets
    if group is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=w.dev)
        t = _allreduce_max(t, group)
        ms = float(t.item())
    tokens = w.cfg.B * w.n_gen if tokens is None else tokens
    return {"value": round(tokens / (ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "steps": steps,
            "pipeline": "uploads of step i+1 (copy stream, double-buffered inputs) overlap step i's compute"}


# ------------------------------------------------------------------------------------------
# the CPU oracle (reference arm / cpu_baseline)
# ------------------------------------------------------------------------------------------
def oracle_sample_time(cfg, tensors):
    """Oracle seconds for a bounded sample of one step: request 0, the last layer,
    one generated token; extrapolated linearly in requests, layers and tokens."""
    import oracle
    vis, txt, K, V, kr, vr, rest_len, q = tensors
    m = cfg.model
    og1 = oracle.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, list(cfg.widths))
    t0 = time.perf_counter()
    sc = oracle.window_scores(vis[:1], txt[:1], cfg.S)
    t1 = time.perf_counter()
    thr = oracle.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    bits, rank, perm, seg = oracle.assign_bits(sc, thr, og1, cfg.budget, 1, 0)
    t2 = time.perf_counter()
    l = cfg.layers - 1
    pk, offs = oracle.reorder_quantize_pack(K[:1], V[:1], 0, og1, perm[l], seg[l])
    t3 = time.perf_counter()
    oracle.decode_attention(q[:1], pk, offs, seg[l], perm[l], og1, kr[:1], vr[:1], rest_len[:1],
                            1 / math.sqrt(m.d))
    t4 = time.perf_counter()
    per = {"scores_1req": t1 - t0, "assign_1req_all_layers": t2 - t1, "quantize_1req_1layer": t3 - t2,
           "decode_1req_1layer_1token": t4 - t3}
    est = (per["scores_1req"] * cfg.B + per["assign_1req_all_layers"] * cfg.B
           + per["quantize_1req_1layer"] * cfg.B * cfg.layers
           + per["decode_1req_1layer_1token"] * cfg.B * cfg.layers * cfg.n_gen)
    return est, per, t4 - t0


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


_ONE_THREAD = r"""
import json, math, sys, time
import numpy as np
sys.path.insert(0, sys.argv[2])
import oracle
z = np.load(sys.argv[1])
S, d, H, Hq = (int(z[k]) for k in ("S", "d", "H", "Hq"))
vis, txt, K, V = z["vis"], z["txt"], z["K"], z["V"]
nw = vis.shape[1] // S
t0 = time.perf_counter()
oracle.window_scores(vis, txt, S)
t1 = time.perf_counter()
M = K.shape[2]
og = oracle.geom(1, H, Hq, d, M, S, [2, 4, 8, 16])
pk, offs = oracle.reorder_quantize_pack(K, V, 0, og, z["perm"], z["seg"])
t2 = time.perf_counter()
oracle.decode_attention(z["q"], pk, offs, z["seg"], z["perm"], og, z["kr"], z["vr"], z["rest_len"], 1 / math.sqrt(d))
t3 = time.perf_counter()
print(json.dumps({"scores_per_window_s": (t1 - t0) / nw, "quantize_1req_1layer_s": t2 - t1,
                  "decode_1req_1layer_1token_s": t3 - t2}))
"""


def oracle_one_thread(cfg, w, l, n_windows=48):
    """The oracle's quantize + decode of one request-layer and its scorer on the first
    n_windows windows, in a child process with OMP_NUM_THREADS=1 (single-core times)."""
    import subprocess
    import tempfile
    m = cfg.model
    S = cfg.S
    with tempfile.TemporaryDirectory() as td:
        f = os.path.join(td, "s.npz")
        np.savez(f, vis=w.vis[:1, :n_windows * S].cpu().numpy(), txt=w.txt[:1].cpu().numpy(),
                 K=w.K[l][:1].cpu().numpy(), V=w.V[l][:1].cpu().numpy(), kr=w.kr[l][:1].cpu().numpy(),
                 vr=w.vr[l][:1].cpu().numpy(), rest_len=w.rest_len[0][:1].cpu().numpy(),
                 q=w.q[0, l][:1].cpu().numpy(), perm=w.perm[l][:1].cpu().numpy(), seg=w.seg[l][:1].cpu().numpy(),
                 S=S, d=m.d, H=m.H, Hq=m.Hq)
        env = dict(os.environ, OMP_NUM_THREADS="1")
        try:
            out = subprocess.run([sys.executable, "-c", _ONE_THREAD, f, ROOT], env=env, capture_output=True,
                                 text=True, timeout=300)
            r = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:
            return {"error": f"{type(e).__name__}: {e}"}
    return {k: round(v, 4) for k, v in r.items()} | {"threads": 1, "scorer_sample_windows": n_windows}


def cpu_baseline(cfg, w, args):
    vis, txt = w.vis[:1].cpu().numpy(), w.txt[:1].cpu().numpy()
    l = cfg.layers - 1
    tensors = (vis, txt, w.K[l][:1].cpu().numpy(), w.V[l][:1].cpu().numpy(), w.kr[l][:1].cpu().numpy(),
               w.vr[l][:1].cpu().numpy(), w.rest_len[0][:1].cpu().numpy(), w.q[0, l][:1].cpu().numpy())
    est, per, wall = oracle_sample_time(cfg, tensors)
    return {"value": round(cfg.B * cfg.n_gen / est, 4), "unit": UNIT, "cores": _cores(), "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": (f"request 0, layer {l}, 1 generated token of {cfg.name} (scores + assign + quantize + decode), "
                       f"{wall:.1f}s of CPU work on {_cores()} threads, extrapolated linearly to B={cfg.B} x "
                       f"{cfg.layers} layers x {cfg.n_gen} tokens"),
            "per_phase_s": {k: round(v, 4) for k, v in per.items()},
            "oracle_1thread": oracle_one_thread(cfg, w, l)}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands on this box's host cores."""
    if rank != 0:
        return None
    import torch
    from paper_2605_02262_b200 import configs, synth
    cfg = configs.CONFIGS[args.config]
    m = cfg.model
    l = cfg.layers - 1
    vis, txt = synth.embeddings(1, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cpu")
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, "cpu", B=1)
    rest_len = rest_len + 1
    q = synth.queries(1, m.Hq, m.H, m.d, cfg.seed, l, 0, "cpu")
    tensors = tuple(t.numpy() for t in (vis, txt, K, V, kr, vr, rest_len, q))
    times = []
    for _ in range(args.warmup):
        oracle_sample_time(cfg, tensors)
    for _ in range(args.steps):
        est, per, wall = oracle_sample_time(cfg, tensors)
        times.append(est)
    ms = float(np.mean(times)) * 1e3
    value = cfg.B * cfg.n_gen / (ms / 1e3)
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1),
            "ms_per_step_kind": (f"extrapolated: each step times a bounded sample ({wall:.1f}s of CPU work) and "
                                 f"scales it linearly to the full step"),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "layers": cfg.layers, "batch": cfg.B, "visual_tokens": cfg.M,
                       "window": cfg.S, "widths": list(cfg.widths), "gen_tokens": cfg.n_gen},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "kind": "oracle", "cores": _cores(),
                             "sample": (f"each step: request 0, layer {l}, 1 token of {cfg.name}; "
                                        f"time extrapolated to the full step"),
                             "cpu_model": _cpu_model()},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wq", choices=["wq", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (profiling only)")
    ap.add_argument("--n-gen", type=int, default=None, help="override generated tokens (profiling only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel from the host (no CUDA graphs)")
    ap.add_argument("--no-ablation", action="store_true", help="skip the T8/T9/T11 ablation measurements")
    ap.add_argument("--parallel", default="auto", choices=["auto", "seqsplit", "batch", "units"],
                    help="N > 1: sequence split (P2, default for C5) or (request, kv-head) unit sharding "
                         "(P1: whole requests, or kv heads of one request; default otherwise)")
    ap.add_argument("--merge", default="peer", choices=["peer", "nccl"],
                    help="N > 1: fused peer-memory LSE merge in the decode kernel, or NCCL all-gather + merge")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        lr = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(lr)
        # WQ_BENCH_BACKEND=gloo: host-side collectives only (testing the P1 batch-sharded
        # mode with several ranks on one GPU; the sequence split needs NCCL / peer memory)
        backend = os.environ.get("WQ_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
        else:
            dist.init_process_group(backend)
    res = run_wq(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
