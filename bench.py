"""Benchmark driver (contract: DESIGN.md section 6).

Headline (BASELINE.json metric "HE images/s (batched)", config 4): the
CIFAR-shaped bi-CryptoNet `cifar3` on 32x32x3 images, N = 2^14, 15 limbs
(max_level = required 13 + 1), Delta = 2^50, BHW packing of 32 images per slot
set; every step runs `forward_bicrypto` over --images images per rank
(default 4096 = 128 slot sets, processed as device batches of --chunk sets)
from plaintext inputs to decrypted logits.  Inputs are far larger than L2
(ciphertext working set: GBs), so no explicit flush is needed.

Parity of the measured configuration: the logits of the LAST timed step (and
of the last end-to-end step) are compared, image by image, with the float64
`reference_forward` (network.py:451-507 restated, pinned to the reference's
golden fixtures) of the very same inputs: max |diff|, argmax agreement.

Also on the line at N = 1: 1-image latency (config 1), the config-2 NTT /
INTT / MAC and config-3 key-switch microbenchmarks, the in-step NTT roofline
(every NTT launch of one forward step timed with CUDA events), the CPU
baseline (the UNMODIFIED reference forward, timed on the host cores) and
CPU-oracle columns for configs 2 and 3.

N > 1: one process per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run), each rank runs its own shard of slot
sets, the logits ciphertexts are gathered to rank 0 (NCCL) and decrypted
there; time = max over ranks.  --workload cfg4: --images per rank (weak
scaling); --workload cfg5: BASELINE config 5, a fixed 65,536-image job split
over the ranks (strong scaling).
`--impl reference`: the reference arm -- the reference's own
`forward_bicrypto` (oracle/_ref, staged by oracle/build_ref.sh) on all host
cores, same metric and workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic  # noqa: E402

IMAGES_PER_SET = 32          # 32 x 16 x 16 = 8192 = N/2 slots
SCALE = 2.0 ** 50
CFG5_IMAGES = 65536
LOGIT_TOL = 1e-6             # absolute, as in tests/test_gpu_network.py
METRIC = "HE images/s (batched)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg5"])
    ap.add_argument("--images", type=int, default=4096, help="cfg4: images per rank per step")
    ap.add_argument("--chunk", type=int, default=128, help="slot sets per device batch")
    ap.add_argument("--no-extras", action="store_true", help="skip latency / micro / cpu baseline")
    ap.add_argument("--ref-seconds", type=float, default=20.0,
                    help="reference arm: target CPU seconds per step (bounded sample)")
    return ap.parse_args()


def cores_available() -> int:
    return len(os.sched_getaffinity(0))


# ----------------------------------------------------------------- workload
def cifar3_weights():
    from paper_2402_01296_b200 import catalog

    bundle = catalog.get("cifar3")
    return bundle, synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.05, seed=3)


def rank_sets(workload: str, images: int, rank: int, world: int) -> range:
    """Slot sets of this rank: cfg4 -- its own `images` (weak scaling);
    cfg5 -- a contiguous shard of the fixed 2048-set job."""
    from paper_2402_01296_b200.shard import shard_range

    if workload == "cfg5":
        return shard_range(CFG5_IMAGES // IMAGES_PER_SET, rank, world)
    return range(-(-images // IMAGES_PER_SET))


def rank_inputs(workload: str, images: int, rank: int, world: int):
    if workload == "cfg5":
        return synthetic.cfg4_set_inputs(rank_sets(workload, images, rank, world))
    return synthetic.cfg4_inputs(images, seed=100 + rank)


def workload_desc(workload: str) -> str:
    base = ("cifar3 bi-CryptoNet, BASELINE config {c}: N=2^14, 15 limbs (q0 + 14 rescale primes, all 50b), "
            "K=5 special 50b, dnum=3, Delta=2^50, BHW 32 images/slot set")
    if workload == "cfg5":
        return base.format(c=5) + f"; fixed {CFG5_IMAGES} images sharded by slot set over the ranks"
    return base.format(c=4)


_REF_JOB: dict = {}


def _ref_logits_job(args_tuple):
    """Worker: float64 reference_forward of a slice of one rank's inputs."""
    import paper_2402_01296_b200 as BCN

    from paper_2402_01296_b200.archive import TensorArchive

    workload, images, rank, world, lo, hi = args_tuple
    key = (workload, images, rank, world)
    if key not in _REF_JOB:                       # per worker process: inputs and weights made once
        _REF_JOB[key] = rank_inputs(workload, images, rank, world)
    if "weights" not in _REF_JOB:
        bundle, w = cifar3_weights()
        _REF_JOB["weights"] = (bundle, TensorArchive(w))
    sens, full = _REF_JOB[key]
    bundle, w = _REF_JOB["weights"]
    return BCN.reference_forward(bundle.bi, synthetic.decomposed(sens[lo:hi], full[lo:hi]), w)


def reference_logits(pool, workload: str, images: int, world: int) -> np.ndarray:
    """reference_forward logits of every rank's inputs, in gather order (rank 0 only)."""
    jobs = []
    for r in range(world):
        n = len(rank_sets(workload, images, r, world)) * IMAGES_PER_SET if workload == "cfg5" else images
        for lo in range(0, n, 256):
            jobs.append((workload, images, r, world, lo, min(n, lo + 256)))
    return np.concatenate(pool.map(_ref_logits_job, jobs))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
        return False

    def summary(self) -> dict:
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def logit_parity(got: np.ndarray, ref: np.ndarray) -> dict:
    err = float(np.abs(got - ref).max())
    agree = float((got.argmax(1) == ref.argmax(1)).mean())
    return {"images_checked": int(got.shape[0]), "max_abs_logit_err": err, "argmax_agreement": agree,
            "tolerance": LOGIT_TOL, "pass": bool(err <= LOGIT_TOL and agree == 1.0)}


# ------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int, dist_on: bool, pool):
    import torch

    import paper_2402_01296_b200 as BCN
    from paper_2402_01296_b200 import _lib, sim
    from paper_2402_01296_b200.archive import TensorArchive
    from paper_2402_01296_b200.shard import gather_to_root

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    bundle, weights = cifar3_weights()
    sens_np, full_np = rank_inputs(args.workload, args.images, rank, world)
    n_img = sens_np.shape[0]
    n_sets_all = sum(len(rank_sets(args.workload, args.images, r, world)) for r in range(world))
    w = TensorArchive(weights)
    ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, SCALE)
    n_sets = -(-n_img // IMAGES_PER_SET)
    chunk_imgs = args.chunk * IMAGES_PER_SET

    sens_d = torch.as_tensor(sens_np, device=dev)
    full_d = torch.as_tensor(full_np, device=dev)
    sens_h = torch.as_tensor(sens_np).pin_memory()
    full_h = torch.as_tensor(full_np).pin_memory()

    # e2e inputs: every step copies its inputs from pinned host memory on a copy
    # stream into one of two device buffers; step k+1's copy is issued when step k
    # starts, so it overlaps step k's compute (each copy is still inside the timed
    # region, and a step waits for its own copy)
    copy_stream = torch.cuda.Stream(device=dev)
    in_bufs = [(torch.empty_like(sens_d), torch.empty_like(full_d)) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for ev in consumed:
        ev.record()

    def issue_copy(slot: int):
        copy_stream.wait_event(consumed[slot])          # the step that last read this buffer is done
        with torch.cuda.stream(copy_stream):
            in_bufs[slot][0].copy_(sens_h, non_blocking=True)
            in_bufs[slot][1].copy_(full_h, non_blocking=True)
            ready[slot].record(copy_stream)

    def step(device_inputs: bool, slot: int = 0):
        outs = []
        if not device_inputs:
            torch.cuda.current_stream().wait_event(ready[slot])
        src = (sens_d, full_d) if device_inputs else in_bufs[slot]
        for s0 in range(0, n_img, chunk_imgs):
            s1 = min(n_img, s0 + chunk_imgs)
            inp = (src[0][s0:s1], src[1][s0:s1])
            res = BCN.forward_bicrypto(bundle.bi, inp, w, ctx, strategy="bhw", group_size=IMAGES_PER_SET)
            outs.append(res)
        return outs

    def run_steps(device_inputs: bool, to_host: bool, n: int):
        last = None
        if not device_inputs:
            issue_copy(0)
        for k in range(n):
            if not device_inputs and k + 1 < n:
                issue_copy((k + 1) % 2)
            last = finish(step(device_inputs, k % 2), to_host)
            if not device_inputs:
                consumed[k % 2].record()
        return last

    def finish(outs, to_host: bool):
        """gather logits ciphertexts to rank 0 and decrypt there."""
        if outs:
            datas = torch.cat([r.logits_ct.data for r in outs])          # (n_sets, 2, 2, N) at level 1
        else:
            datas = torch.zeros((0, 2, 2, 1 << 14), dtype=torch.int64, device=dev)
        if dist_on:
            datas = gather_to_root(datas, n_sets_all)
        if rank != 0:
            return None
        slots = ctx.engine.decrypt(datas, 1, SCALE)
        idx = torch.arange(IMAGES_PER_SET, device=dev)[:, None] * outs[0].tile_step + torch.arange(10, device=dev)
        logits = slots[:, idx].reshape(-1, 10)
        return logits.cpu() if to_host else logits

    def timed(device_inputs: bool, to_host: bool, K: int, W: int, rec_clocks: bool):
        run_steps(device_inputs, to_host, W)
        if dist_on:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        l0 = _lib.launch_count()
        cs = ClockSampler(dev.index) if rec_clocks else None
        if cs:
            cs.__enter__()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("timed_e2e" if to_host else "timed")   # ncu --nvtx-include timed/
        s.record()
        last = run_steps(device_inputs, to_host, K)
        e.record()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        if cs:
            cs.__exit__()
        if dist_on:
            torch.distributed.barrier()
        ms = s.elapsed_time(e) / K
        if dist_on:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, (_lib.launch_count() - l0) // K, cs.summary() if cs else None, last

    # reference counts and device work of one forward (recorder == the reference's integers)
    sim.reset_stats()
    rec_res = BCN.forward_bicrypto(bundle.bi, (sens_d[:IMAGES_PER_SET], full_d[:IMAGES_PER_SET]), w, ctx,
                                   strategy="bhw", group_size=IMAGES_PER_SET)
    counts = rec_res.recorder.snapshot()
    dev_work = dict(sim.STATS)

    keys_agree = None
    if dist_on:
        # keys are regenerated on every rank from the shared seed (no broadcast);
        # check it once with a key-checksum all-gather
        k = ctx.engine.export_key(2)
        h = torch.stack([k.sum(), (k * torch.arange(1, k.shape[-1] + 1, device=k.device)).sum()])
        hs = [torch.empty_like(h) for _ in range(world)]
        torch.distributed.all_gather(hs, h)
        keys_agree = all(bool((x == hs[0]).all()) for x in hs)
        if not keys_agree:
            raise RuntimeError("switching keys differ across ranks")

    # float64 reference logits of every image this job decrypts (CPU pool, before timing)
    ref_all = reference_logits(pool, args.workload, args.images, world) if rank == 0 else None

    ms, launches, clocks, last = timed(True, False, args.steps, args.warmup, True)
    total_images = n_sets_all * IMAGES_PER_SET if args.workload == "cfg5" else args.images * world
    value = total_images / (ms / 1e3)
    e2e_ms, _, _, last_e2e = timed(False, True, args.steps, max(1, args.warmup // 3), False)
    e2e = total_images / (e2e_ms / 1e3)

    parity = None
    if rank == 0:
        parity = {"timed_step": logit_parity(last.cpu().numpy()[:total_images], ref_all),
                  "timed_e2e_step": logit_parity(last_e2e.numpy()[:total_images], ref_all),
                  "reference": "reference_forward (float64 clear forward, network.py:451-507 restated; pinned to "
                               "the reference's golden fixtures in tests/test_host.py)",
                  "counts_per_forward": counts}
    # in-step NTT roofline: one more (untimed) step with every NTT launch bracketed by CUDA events
    ntt_step = conv_step = None
    if rank == 0 and world == 1:
        torch.cuda.synchronize()
        _lib.ntt_timing(True)
        _lib.conv_timing(True)
        finish(step(True), False)
        torch.cuda.synchronize()
        _lib.ntt_timing(False)
        _lib.conv_timing(False)
        ntt_step = _lib.ntt_timing_read()
        conv_step = _lib.conv_timing_read()
    h2d = sens_np.nbytes + full_np.nbytes
    d2h = total_images * 10 * 8 if rank == 0 else 0
    return {
        "value": value, "ms_per_step": ms, "e2e": {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": h2d,
                                                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                                                    "note": "every step copies its inputs from pinned host memory "
                                                            "(copy stream, double buffer: step k+1's copy overlaps "
                                                            "step k) and reads its logits back to the host"},
        "gpu_launches": launches, "clocks": clocks, "counts_per_forward": counts, "keys_agree_across_ranks": keys_agree,
        "device_work_per_forward": dev_work, "parity": parity, "ctx": ctx, "ntt_step": ntt_step,
        "conv_step": conv_step,
        "total_images": total_images,
    }


def latency_cfg1(reps: int = 10):
    """Config 1: one 28x28 image, cnn3, N=2^13, 11 limbs; host -> host."""
    import torch

    import paper_2402_01296_b200 as BCN
    from paper_2402_01296_b200.archive import TensorArchive
    from paper_2402_01296_b200.network import DecomposedInput

    bundle = BCN.get("cnn3")
    w = TensorArchive(synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.1, seed=1))
    sens, full = synthetic.cfg1_inputs(1, seed=0)
    dec = [DecomposedInput(sens[0], full[0], (7, 7, 14, 14))]
    ctx = BCN.make_context(8192, BCN.required_levels(bundle) + 1, SCALE)
    for _ in range(3):
        BCN.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="hw").decrypt_logits()
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        BCN.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="hw").decrypt_logits()
        times.append(time.perf_counter() - t0)
    ref = BCN.reference_forward(bundle.bi, dec, w)
    got = BCN.forward_bicrypto(bundle.bi, dec, w, ctx, strategy="hw").decrypt_logits()
    # the serving path: the whole request (H2D inputs, encrypt, forward, decrypt, D2H) as one CUDA graph
    from paper_2402_01296_b200.graphs import GraphedForward
    gf = GraphedForward(bundle.bi, w, ctx, sens.shape, full.shape, strategy="hw")
    sens_h = torch.as_tensor(sens).pin_memory()
    full_h = torch.as_tensor(full).pin_memory()
    for _ in range(3):
        gf(sens_h, full_h)
    gtimes = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g_logits = gf(sens_h, full_h)
        gtimes.append(time.perf_counter() - t0)
    gf.close()
    return {"metric": "1-image latency (cnn3, config 1)", "value": statistics.median(gtimes), "unit": "s",
            "path": "CUDA-graph replay (GraphedForward), host inputs -> host logits",
            "eager_value": statistics.median(times), "reps": reps,
            "max_abs_logit_err": float(max(np.abs(got - ref).max(), np.abs(g_logits - ref).max())),
            "paper_SEAL_cpu_latency_s": 2.1}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def ntt_roofline(ntt_step: dict, peak: float, peak_kind: str) -> dict:
    """Byte-weighted roofline fraction of ALL NTT/INTT launches of one forward step
    (the NTT family is the largest share of the step, profiles/)."""
    tot_b = sum(v["bytes"] for v in ntt_step.values())
    tot_ms = sum(v["ms"] for v in ntt_step.values())
    achieved = tot_b / (tot_ms * 1e-3) / 1e9 if tot_ms else 0.0
    per = {k: dict(v, GBps=(v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else None),
                   frac=(v["bytes"] / (v["ms"] * 1e-3) / 1e9 / peak if v["ms"] else None))
           for k, v in ntt_step.items()}
    return {
        "kernel": "NTT/INTT family (ntt_fwd_cluster<14,*>, ntt_inv_cluster<14>): every launch of one cifar3 "
                  "forward step (4096 images), byte-weighted; class encrypt_fwd is the encryption's forward NTT "
                  "with c0 = NTT(m+e) - a s and c1 = a (Philox) computed in its epilogue",
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "peak_kind": peak_kind, "traffic": _traffic().get("ntt14_fwd"),
        "algorithmic_bytes_per_step": tot_b, "ntt_ms_per_step": tot_ms,
        "algorithmic_bytes_per_unit": "16 B per coefficient of each limb-poly transformed (one u64 read + one u64 "
                                      "write) plus the operands a fused prologue/epilogue reads once (rescale-lift "
                                      "top limb per poly, combine inputs c/A/B, ModDown addend sigma(c0), "
                                      "epilogue-4 U digits); keys and twiddles excluded (csrc/ntt.cu "
                                      "ntt_algorithmic_bytes)",
        "launches": sum(v["launches"] for v in ntt_step.values()), "by_class": per,
        "timing": "CUDA event pair around every NTT launch on its stream (bcn_ntt_timing), one untimed step "
                  "after the timed region"}


def conv_roofline(conv_step: dict, peak: float, step_ms: float) -> dict:
    """The conv operand path of one forward step on the HBM roof: every slot-major staging launch
    (slot_major_ks3 with the key-switch inner products, slot_major for the pre-rotated first conv) and
    every tensor-core MAC launch (mac_umma), from a CUDA event pair around each (bcn_conv_timing)."""
    out = {}
    for k, v in conv_step.items():
        gbps = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else None
        out[k] = dict(v, GBps=gbps, frac=(gbps / peak if gbps else None), share_of_step=v["ms"] / step_ms)
    out["algorithmic_bytes_per_launch"] = (
        "staging: each distinct source's U digits, c0 and c1 and each term's key words once + the staged words "
        "written (8 B x slots x terms x 2 x slot sets per limb); MAC: the staged words read once + the plaintext "
        "byte planes + the outputs written (csrc/api.cu bcn_conv_ks_mac / bcn_mac_multi_planes_layout)")
    return out


# ------------------------------------------------------------ CPU columns
def cpu_reference_forward(cores: int, weights: dict, target_s: float, steps: int = 2, warmup: int = 0) -> dict:
    """The UNMODIFIED reference forward_bicrypto (oracle/_ref) on `cores` worker
    processes over independent BHW-32 slot sets of config-4 images."""
    from oracle import ref_arm

    sens, full = synthetic.cfg4_inputs(cores * IMAGES_PER_SET * (steps + warmup + 1), seed=100)
    ref_arm.setup(weights, sens, full, backend="")
    return ref_arm.time_forward(cores, steps, warmup)


def ks_compute_bound(c3: dict, n14: dict) -> dict:
    """Compute-aware floor of config 3 next to its HBM fraction (SURVEY.md
    8(d)'s compute reference): limb-transforms x the N = 2^14 NTT time per
    limb-poly measured in this run (bench_micro.ntt14), plus the inner
    products at the measured 64-bit MAC rate of the IMAD pipe (Acc4, 5.5
    MAC/clk/SM, tools/micro/mac_bench.cu).  Per key switch at level l with
    l+1 = 8 limbs, K = 1, alpha = 4, dnum = 2: ModUp = (l+1) INTT + dnum (l+1+K-alpha)
    NTT; ModDown = 2K INTT + 2(l+1) NTT; inner product 2 dnum (l+1+K) N MACs.
    Stage A: 1024 full key switches; stage B: 1024 ModUps + 14 x 1024
    (inner product + ModDown)."""
    n_ct, limbs, K, alpha, dnum, N, rots = 1024, 8, 1, 4, 2, 16384, 14
    us_fwd = n14["fwd"]["ms"] * 1e3 / n14["limb_polys"]
    us_inv = n14["inv"]["ms"] * 1e3 / n14["limb_polys"]
    modup = limbs * us_inv + dnum * (limbs + K - alpha) * us_fwd
    moddown = 2 * K * us_inv + 2 * limbs * us_fwd
    mac_rate = 5.5 * 148 * 1.965e9                      # 64-bit modular MACs / s
    inner_ms = 2 * dnum * (limbs + K) * N / mac_rate * 1e3
    a_ms = n_ct * (modup + moddown) / 1e3 + n_ct * inner_ms
    b_ms = n_ct * modup / 1e3 + n_ct * rots * (moddown / 1e3 + inner_ms)
    return {"relin": {"bound_ms": a_ms, "measured_ms": c3["relin"]["ms"], "frac": a_ms / c3["relin"]["ms"]},
            "rotations": {"bound_ms": b_ms, "measured_ms": c3["rotations"]["ms"],
                          "frac": b_ms / c3["rotations"]["ms"]},
            "ntt_us_per_limb_poly": {"fwd": us_fwd, "inv": us_inv},
            "limb_transforms": {"relin_per_ct": limbs + dnum * (limbs + K - alpha) + 2 * K + 2 * limbs,
                                "rotations_per_ct": limbs + dnum * (limbs + K - alpha) + rots * (2 * K + 2 * limbs)},
            "note": "floor = NTT limb-transforms at this run's measured us/limb-poly + inner-product MACs at "
                    "the IMAD-pipe rate; frac = floor / measured"}


def cpu_oracle_columns() -> dict:
    """Configs 2 and 3 have no reference counterpart (the reference does no
    cryptography): the C/numpy RNS-CKKS oracle port on the same shapes, on a
    stated subsample, scaled linearly.  kind "port"."""
    from oracle import ckks as O

    out = {}
    # config 2: NTT / INTT of 256 of the 32,768 limb-polys (N = 8192, 60-bit primes), MAC of 2 groups of 25
    p2 = O.make_params(8192, 3, 60, dnum=1, n_special=1)
    rng = np.random.default_rng(0)
    sub = 256
    x = np.stack([rng.integers(0, p2.q[i % 4], 8192, dtype=np.uint64) for i in range(sub)])
    t0 = time.perf_counter()
    for i in range(4):
        O.ntt_batch(x[i::4].copy(), p2.q[i])
    t_ntt = time.perf_counter() - t0
    t0 = time.perf_counter()
    for i in range(4):
        O.intt_batch(x[i::4].copy(), p2.q[i])
    t_intt = time.perf_counter() - t0
    cts = [np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in p2.q]) for _ in range(2 * 25)]
    pts = [np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in p2.q]) for _ in range(25)]
    t0 = time.perf_counter()
    for g in range(2):                       # 2 output groups x 25 terms x 2 components
        acc = np.zeros_like(cts[0])
        for t in range(25):
            for c in range(2):
                acc = O.add(acc, O.mul(cts[(g * 25 + t) % 50], pts[t], p2.q), p2.q)
    t_mac = (time.perf_counter() - t0) / 2 * 164
    scale = 32768 / sub
    # config 2 fused (NTT -> MAC -> rescale, oracle.ntt_mac_rescale) on 2 of the 164 groups, u64 and u32 primes
    fused = {}
    for tag, bits in (("u64", 60), ("u32", 30)):
        primes = O.ntt_primes(bits, 4, 8192)
        fc = np.stack([np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in primes])
                                 for _ in range(2)]) for _ in range(50)])
        fp = np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in primes]) for _ in range(50)])
        t0 = time.perf_counter()
        O.ntt_mac_rescale(fc, fp, primes, 25)
        fused[tag + "_ms"] = (time.perf_counter() - t0) / 2 * 164 * 1e3
    out["config2"] = {**{"fused_" + k: v for k, v in fused.items()}, "ntt_ms": t_ntt * scale * 1e3, "intt_ms": t_intt * scale * 1e3, "mac_ms": t_mac * 1e3,
                      "sample": f"{sub} of 32768 limb-polys (NTT/INTT), 2 of 164 MAC groups, 2 of 164 fused "
                                "NTT+MAC+rescale groups (u64: 60-bit, u32: 30-bit primes); scaled linearly",
                      "kind": "port", "cores": int(os.environ.get("OMP_NUM_THREADS", cores_available()))}
    # config 3: one ct x ct + relinearisation (merged with rescale) and 2 of the 14 hoisted rotations of one
    # ciphertext (N = 16384, 8 limbs, K = 1, dnum = 2); scaled to 1024 ciphertexts x 14 rotations
    p3 = O.make_params(16384, 7, 50, dnum=2, n_special=1)
    orc = O.Oracle(p3)
    v = rng.standard_normal(8192) * 0.1
    ct = orc.encrypt(v, 1)
    orc.relin_key()
    g1, g2 = O.galois_elt(1, 16384), O.galois_elt(-1, 16384)
    orc.galois_key(g1)
    orc.galois_key(g2)
    t0 = time.perf_counter()
    orc.mul_cc(ct, ct)
    t_relin = time.perf_counter() - t0
    t0 = time.perf_counter()
    U = orc.modup(ct.c1, 7)
    for g in (g1, g2):
        orc.keyswitch_from_modup(U, 7, orc.galois_key(g), g)
    t_rot = time.perf_counter() - t0
    out["config3"] = {"relin_ms": t_relin * 1024 * 1e3, "rotations_ms": t_rot / 2 * 14 * 1024 * 1e3,
                      "sample": "1 of 1024 squarings (+relinearise), 2 of 14 rotations of 1 of 1024 ciphertexts "
                                "(shared ModUp); scaled linearly",
                      "kind": "port", "cores": int(os.environ.get("OMP_NUM_THREADS", cores_available()))}
    return out


# ------------------------------------------------------------ reference arm
def run_reference(args) -> None:
    """The reference's own forward_bicrypto on all host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from oracle import ref_arm

    if not ref_arm.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not staged (run oracle/build_ref.sh)"}))
        return
    cores = cores_available()
    _, weights = cifar3_weights()
    # one step = `cores` slot sets in parallel (~0.35-0.6 s each); enough steps per timed step for
    # a bounded sample of about --ref-seconds of CPU work in total per step
    groups_per_core = max(1, int(round(args.ref_seconds / cores / 0.45)))
    total_groups = cores * groups_per_core
    sens, full = synthetic.cfg4_inputs(min(4096, total_groups * IMAGES_PER_SET), seed=100)
    ref_arm.setup(weights, sens, full, backend="")
    import multiprocessing as mp
    per_step = []
    with mp.get_context("fork").Pool(cores, initializer=ref_arm._worker_init) as pool:
        pool.map(ref_arm.group_forward, range(cores))
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(ref_arm.group_forward, range(i * total_groups, (i + 1) * total_groups))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                per_step.append(dt)
    images = total_groups * IMAGES_PER_SET
    value = images * len(per_step) / sum(per_step)
    line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(per_step),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded cfg4 images, N(0,0.05) weights)", "impl": "reference",
            "config": {"workload": workload_desc("cfg4"), "images_per_step": images,
                       "note": "reference simulator, no cryptography (sim.py:1-12)"},
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "reference",
                             "sample": f"{images} config-4 images per step = {total_groups} BHW-32 slot sets "
                                       f"through the unmodified reference forward_bicrypto "
                                       f"(network.py:388-448, {ref_arm._ST['R'].active_backend()} slot kernels), "
                                       f"{cores} worker processes, one thread each"},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ main
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(args) -> int:
    """`--gpus N` outside torchrun: launch N ranks (one per GPU) of this script."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        sys.exit(relaunch_distributed(args))
    world = int(world_env or 1)
    rank = int(os.environ.get("RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    dist_on = world > 1
    # CPU pool for the float64 reference logits, forked before any CUDA call
    import multiprocessing as mp
    pool = mp.get_context("fork").Pool(max(1, min(16, cores_available()))) if rank == 0 else None
    import torch

    if dist_on:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        res = run_ours(args, rank, world, dist_on, pool)
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    extras = {}
    if rank == 0 and not args.no_extras and world == 1:
        import bench_micro
        extras["latency_1img"] = latency_cfg1()
        c2 = bench_micro.config2()
        c2f = bench_micro.config2_fused()
        c3 = bench_micro.config3()
        n14 = bench_micro.ntt14()
        extras["micro"] = {"config2": c2, "config2_fused": c2f, "config3": c3, "ntt14": n14,
                           "ks_bound": ks_compute_bound(c3, n14)}
        peak, peak_kind = _peaks()
        extras["roofline"] = ntt_roofline(res["ntt_step"], peak, peak_kind)
        extras["roofline_conv"] = conv_roofline(res["conv_step"], peak, res["ms_per_step"])
        extras["roofline_micro"] = {
            "ntt14_fwd": {"achieved": n14["fwd"]["GBps"], "frac": n14["fwd"]["GBps"] / peak,
                          "launch": "ntt_fwd_cluster<14,0,0>, 1536 limb-polys, 1 launch"},
            "ntt14_inv": {"achieved": n14["inv"]["GBps"], "frac": n14["inv"]["GBps"] / peak}}
        for name in ("ntt", "intt", "mac"):
            extras["roofline_micro"]["cfg2_" + name] = {"achieved": c2[name]["GBps"], "frac": c2[name]["GBps"] / peak}
        for name in ("relin", "rotations"):
            extras["roofline_micro"]["ks_" + name] = {"achieved": c3[name]["GBps"], "frac": c3[name]["GBps"] / peak}
        for name in ("u64", "u32", "u32_ntt", "u32_intt"):
            extras["roofline_micro"]["cfg2_fused_" + name] = {"achieved": c2f[name]["GBps"],
                                                              "frac": c2f[name]["GBps"] / peak}
        _, weights = cifar3_weights()
        cores = cores_available()
        cpu = cpu_reference_forward(cores, weights, 20.0)
        extras["cpu_baseline"] = {
            "value": cpu["images_per_s"], "unit": "images/s", "cores": cores, "kind": "reference",
            "sample": f"2 steps x {cpu['images_per_step']} config-4 images (one BHW-32 slot set per worker) through "
                      f"the unmodified reference forward_bicrypto (oracle/_ref, {cpu['backend']} slot kernels): "
                      "reference simulator, no cryptography",
            "seconds_per_step": cpu["seconds_per_step"]}
        extras["cpu_oracle_port"] = cpu_oracle_columns()
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "strong" if args.workload == "cfg5" else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded cfg4 images, N(0,0.05) weights)",
            "config": {"workload": workload_desc(args.workload), "images_per_step": res["total_images"],
                       "slot_sets_per_device_batch": args.chunk,
                       "l2": "working set >> 126 MB L2 (no flush needed)"},
            "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
            "parity": dict(res["parity"], keys_agree_across_ranks=res["keys_agree_across_ranks"]),
            "device_work_per_forward": res["device_work_per_forward"],
        }
        line.update(extras)
        print(json.dumps(line))
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
