#!/usr/bin/env python
"""Batched TFHE programmable bootstrapping on B200 -- BASELINE.json config 2.

One step = one PBS pass (mod switch -> 630-step CMUX-ladder blind rotation ->
sample extraction -> LWE key switch) over a batch of 4096 LWE ciphertexts
(n = 630, N = 1024, l = 3, Bg = 2^7, KS 2^2 x 8, q = 2^32), messages uniform in
Z_8, LUT = identity on [0, 4) with the negacyclic sign on [4, 8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hwb|reference]

Prints ONE JSON line (rank 0).  `value` = whole-job PBS/s with inputs resident
in HBM; `e2e` = the same through the public API from pinned host buffers with
H2D/D2H inside the timed region.  `--impl reference` times the CPU port of the
reference algorithm (oracle/c, all host threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

# FFT ladder mode (hwb_set_fft_mode) -> the kernel that runs a cfg2 batch of 4096
FFT_KERNELS = {0: "blind_rotate_fft_kernel", 1: "blind_rotate_fft_tm_kernel", 2: "blind_rotate_fft_tx_kernel",
               3: "blind_rotate_fft_tp_kernel", 4: "blind_rotate_fft_tq_kernel", 5: "blind_rotate_fft_td_kernel",
               6: "blind_rotate_fft_td_kernel<4,2>", 7: "blind_rotate_fft_w_kernel", 8: "blind_rotate_fft_td_kernel"}
METRIC = "bootstrappings/sec"
UNIT = "PBS/s"
KEY_SEED, ENC_SEED = 1, 2
L2_FLUSH_BYTES = 512 << 20          # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hwb", "reference"], default="hwb")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--ladder", default="auto", choices=["auto", "fft", "ntt"],
                    help="blind rotation: FP64 FFT ladder or two-prime NTT ladder (bit-identical)")
    ap.add_argument("--fft-mode", type=int, default=5, choices=list(range(7)),
                    help="FFT ladder (bit-identical): 0 register accumulators; TMEM accumulators with "
                         "1 two ciphertexts per thread, 2 one per thread, 3 lane-paired, 4 one 16-warp CTA, "
                         "5 lane-paired decoupled halves (default), 6 = 5 as one 16-warp CTA with a 2-slot key ring")
    ap.add_argument("--ks-engine", default="auto", choices=["auto", "tc", "simt"],
                    help="LWE key switch: tensor cores (tcgen05 int8) or the integer-pipe kernel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="PBS per CPU step (0 = auto)")
    ap.add_argument("--train-cfg", type=int, default=3, choices=[1, 3, 4, 5])
    ap.add_argument("--train-images", type=int, default=128, help="0 disables the training measurement")
    ap.add_argument("--train-batch", type=int, default=32)
    ap.add_argument("--infer-images", type=int, default=32, help="0 disables the inference measurement")
    ap.add_argument("--infer-pbs-images", type=int, default=4,
                    help="images for the fully encrypted bleach/popcount/argmax inference (0 disables)")
    ap.add_argument("--infer-pbs-thr", type=int, default=0, help="bleaching threshold of that inference")
    ap.add_argument("--cfg4-train", type=int, default=16384, help="cfg4 full-size variant: training images")
    ap.add_argument("--cfg4-test", type=int, default=2048, help="cfg4 full-size variant: PD-act test images")
    ap.add_argument("--cfg4-pbs-images", type=int, default=2, help="cfg4 variant: fully encrypted inference images")
    ap.add_argument("--no-cfg4-full", dest="cfg4_full", action="store_false", help="skip the full-size cfg4 run")
    ap.add_argument("--no-other-configs", dest="other_configs", action="store_false",
                    help="skip the cfg1/cfg4 PBS measurements")
    ap.add_argument("--sweep", default="1,16,148,592,1184,4096,16384,65536",
                    help="comma-separated PBS batch sizes for the cfg2 sweep ('' disables)")
    return ap.parse_args()


def workload(P, B, rank):
    from paper_2403_20190_b200 import tfhe
    keys = tfhe.pbs_keygen(P, KEY_SEED)
    rng = tfhe.make_rng(ENC_SEED + 1000 * rank)
    ms = rng.integers(0, P.p, B)
    lwe = tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng)
    tv = tfhe.test_polynomial(np.arange(P.p // 2), P)
    return keys, ms, lwe, tv


def expected(ms, p):
    half = p // 2
    return np.where(ms < half, ms, (-(ms - half)) % p)


def config(P, B, world, extra=None):
    c = {"workload": "cfg2 batched PBS (BASELINE.json configs[1])", "batch_per_gpu": B,
         "global_batch": B * world, "n": P.lwe_n, "N": P.n, "k": 1,
         "pbs_gadget": f"Bg=2^{P.gadget.base_log} l={P.gadget.levels}",
         "ks_gadget": f"2^{P.gadget_ks.base_log} l={P.gadget_ks.levels}",
         "q": "2^32", "p": P.p, "lut": "identity on [0,4), negacyclic sign on [4,8)",
         "parallelism": f"replicas{world}" if world > 1 else "single",
         "l2": "flushed (512 MiB write) before every timed step"}
    if extra:
        c.update(extra)
    return c


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_cpu_port(P, keys, lwe, tv, sample, threads):
    """The oracle port (oracle/c, exact schoolbook restatement of the reference
    path) on `sample` ciphertexts; returns (PBS/s, outputs)."""
    from oracle import coracle
    coracle.build()
    t0 = time.perf_counter()
    out = coracle.pbs(lwe[:sample], tv, keys.bsk, keys.ksk, P, nthreads=threads)
    dt = time.perf_counter() - t0
    return sample / dt, out


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "samples": len(rows), "reasons": reasons}


def probe_modmul_peak(torch, _lib, tfhe):
    """Measured P_mm: register-only RNS modmul throughput (one launch filling
    every SM), best of 3, CUDA events on the launching stream."""
    import ctypes
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    L = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 2048
    best = 0.0
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = L.hwb_probe_modmul(ctypes.c_void_p(sink.data_ptr()), blocks, iters, tfhe._stream())
        e.record()
        e.synchronize()
        if n < 0:
            raise RuntimeError(L.hwb_last_error().decode())
        best = max(best, n / (s.elapsed_time(e) * 1e-3))
    return best


def ncu_traffic(B, alg_bytes=None, ladder="ntt"):
    """DRAM bytes per blind-rotation launch from the committed ncu --set full
    capture (profiles/ncu_traffic.json) when it was taken at this batch size."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            rec = json.load(f)[ladder if ladder.startswith("blind_rotate_fft") else "blind_rotate_kernel<1024,PBS>"]
    except (OSError, KeyError, ValueError):
        return None
    if rec.get("batch") != B:
        return None
    return {"bytes": int(rec["dram_bytes_read"] + rec["dram_bytes_write"]), "unit": "B per PBS batch",
            "algorithmic_bytes": alg_bytes, "source": rec.get("source")}


def probe_fp64_peak(torch, _lib, tfhe):
    """Measured P_fp64: register-only DFMA throughput (one launch filling every SM),
    best of 4, CUDA events on the launching stream."""
    import ctypes
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    L = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    best = 0.0
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = L.hwb_probe_fp64(ctypes.c_void_p(sink.data_ptr()), sms * 8, 1024, tfhe._stream())
        e.record()
        e.synchronize()
        if n < 0:
            raise RuntimeError(L.hwb_last_error().decode())
        best = max(best, n / (s.elapsed_time(e) * 1e-3))
    return best


def probe_i8mma_peak(torch, _lib, tfhe):
    """Measured P_i8: tcgen05.mma kind::i8 MAC rate of the key switch's MMA shape
    (M128 N256 K32 from shared memory, one CTA per SM), best of 4."""
    import ctypes
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    L = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    best = 0.0
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = L.hwb_probe_i8mma(ctypes.c_void_p(sink.data_ptr()), sms, 4096, tfhe._stream())
        e.record()
        e.synchronize()
        if n < 0:
            raise RuntimeError(L.hwb_last_error().decode())
        best = max(best, n / (s.elapsed_time(e) * 1e-3))
    return best


def train_other(cfg, images, batch, rank, torch):
    """Device-resident he_train throughput of another BASELINE training config
    (images/s), with the decrypted-counter check where q = 2^32 can decrypt."""
    from paper_2403_20190_b200 import data, hewnn, tfhe, wnn
    from paper_2403_20190_b200.params import named_params
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[cfg]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    ds = data.config_dataset(cfg, n=images, seed=rank)
    key = tfhe.SecretKey(P, tfhe.make_rng(KEY_SEED).integers(0, 2, P.n).astype(np.uint32))
    rng = tfhe.make_rng(ENC_SEED + 2000 + 1000 * rank)
    samples = [hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits,
                                    device=True) for i in range(images)]
    hewnn.he_train(samples[:batch], geom, P, batch=batch)                    # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    model = hewnn.he_train(samples, geom, P, batch=batch)
    e1.record()
    e1.synchronize()
    out = {"images_per_s": round(images / (e0.elapsed_time(e1) * 1e-3), 2), "images": images, "batch": batch,
           "params": f"{pname} N={P.n} Bg=2^{P.gadget.base_log} l={P.gadget.levels}",
           "geometry": {"s": s, "l": l, "a": a, "k0": geom.k0},
           "ladder": "fp64 FFT" if hewnn._use_fft(P, "auto") else "two-prime NTT"}
    if P.p * 2 <= P.n or cfg != 4:
        dm, cc = hewnn.decrypt_model(model, key)
        ref, rc = wnn.train_integer(ds.bits, ds.labels, geom)
        out["check"] = ("decrypted counters == train_integer"
                        if np.array_equal(dm.counters, ref.counters) and np.array_equal(cc.counts, rc.counts)
                        else "COUNTER MISMATCH")
    else:
        out["check"] = "not decryptable at q = 2^32 (p = 4096, DESIGN.md §6b); bit-exactness is tested"
    return out


def bench_train(args, world, rank, torch, dist):
    """Encrypted WiSARD training throughput (the metric's second half):
    hewnn.he_train over `--train-images` client-encrypted images of BASELINE
    config `--train-cfg` (default 3), inputs device-resident (value) and from
    pinned host memory with H2D/D2H inside the timed region (e2e)."""
    from paper_2403_20190_b200 import data, hewnn, tfhe, wnn
    from paper_2403_20190_b200.params import named_params
    cfg, images, batch = args.train_cfg, args.train_images, args.train_batch
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[cfg]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    ds = data.config_dataset(cfg, n=images, seed=rank)
    key = tfhe.SecretKey(P, tfhe.make_rng(KEY_SEED).integers(0, 2, P.n).astype(np.uint32))
    rng = tfhe.make_rng(ENC_SEED + 1000 * rank)
    # client: seeded encryption -- host draws the normals only, the GPU regenerates the
    # uniform a-halves from the Philox stream and forms b; the wire form is b + seeds
    t0 = time.perf_counter()
    seeded = [hewnn.encrypt_sample_seeded(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits)
              for i in range(images)]
    torch.cuda.synchronize()
    enc_s = time.perf_counter() - t0
    samples = [hewnn.EncryptedSample.from_stack(P, x.rgsw.expand(), x.s, x.n_label_bits) for x in seeded]
    hewnn.he_train(samples[:batch], geom, P, batch=batch)                    # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    model = hewnn.he_train(samples, geom, P, batch=batch)
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dm, cc = hewnn.decrypt_model(model, key)
    ref, rc = wnn.train_integer(ds.bits, ds.labels, geom)
    ok = bool(np.array_equal(dm.counters, ref.counters) and np.array_equal(cc.counts, rc.counts))
    noise, margin = hewnn.model_noise(model, key)
    frac_ok = float(np.mean(dm.counters == ref.counters))
    # end to end from the pinned host wire form (b halves + Philox states), model read back
    host = seeded
    h2d = sum(int(h.rgsw.b.numel() + h.rgsw.a0.numel()) * 4 + 80 * len(h.rgsw.segments) for h in host)
    rams_pin = torch.empty(model.rams.shape, dtype=torch.int32).pin_memory()
    del samples
    # warm the pinned-host pipeline once (two chunks in flight: the staging and table
    # buffers it needs are allocated here, not inside the timed region)
    hewnn.he_train(host[: 2 * batch], geom, P, batch=batch)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    m2 = hewnn.he_train(host, geom, P, batch=batch)
    rams_pin.copy_(m2.rams, non_blocking=True)
    f1.record()
    f1.synchronize()
    te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    k1 = hewnn.model_row_polys(geom, P)
    lb = geom.label_bits
    ext_per_img = geom.k0 * (min(lb + geom.a, P.degree_log) + (1 << max(0, lb + geom.a - P.degree_log)) - 1) + lb
    out = {"metric": "encrypted train images/sec", "unit": "images/s",
           "value": round(images * world / (float(t.item()) * 1e-3), 2),
           "config": {"workload": f"BASELINE cfg{cfg} encrypted WiSARD training (he_train)",
                      "params": pname, "p": p, "geometry": {"s": s, "l": l, "a": a, "r": r, "k0": geom.k0,
                                                            "k1": k1}, "images_per_gpu": images,
                      "batch_images": batch, "ext_products_per_image": ext_per_img,
                      "data": "synthetic (data.config_dataset)"},
           "e2e": {"value": round(images * world / (float(te.item()) * 1e-3), 2), "unit": "images/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(model.rams.numel()) * 4,
                   "api": "hewnn.he_train from pinned host seeded RGSW stacks (b halves + Philox states; "
                          "the GPU regenerates a), model read back"},
           "client_encrypt_s_per_image": round(enc_s / images, 4),
           "noise": {"max_log2": round(float(np.log2(max(noise, 1))), 2),
                     "margin_log2": round(float(np.log2(margin)), 2), "counters_correct": round(frac_ok, 6)},
           "check": "decrypted counters == train_integer" if ok else "COUNTER MISMATCH"}
    if args.infer_images > 0:
        # PD-act inference (hw/hewnn.py:278-345) with the trained model
        tds = data.config_dataset(cfg, split="test", n=args.infer_images, seed=rank)
        _, pksk = tfhe.keygen(P, KEY_SEED)                       # same S1 as `key` (first draw)
        trng = tfhe.make_rng(ENC_SEED + 7 + 1000 * rank)
        tsamples = [hewnn.encrypt_sample(tds.bits[i], None, key, trng) for i in range(args.infer_images)]
        pksk.spectra()
        hewnn.he_infer_pd_batch(model, tsamples[:1], pksk)                 # warm-up
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        packs = hewnn.he_infer_pd_batch(model, tsamples, pksk)
        g1.record()
        g1.synchronize()
        act = wnn.ActivationSpec("bin", 0)
        preds = [hewnn.client_finalize(pk, key, act).prediction for pk in packs]
        plain = wnn.evaluate_dataset(ref, tds.bits, act)
        vp_items = geom.l * geom.k0
        out["infer"] = {"metric": "encrypted inference images/sec", "unit": "images/s",
                        "value": round(args.infer_images / (g0.elapsed_time(g1) * 1e-3), 2),
                        "images": args.infer_images, "vp_items_per_image": vp_items,
                        "packed_rlwe_per_image": -(-vp_items // P.n),
                        "check": "predictions == plaintext evaluate" if list(plain) == preds
                        else "PREDICTION MISMATCH"}
        if args.infer_pbs_images > 0:
            out["infer_pbs"] = bench_infer_pbs(args, model, key, ref, tsamples[: args.infer_pbs_images],
                                               tds.bits[: args.infer_pbs_images], torch)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import coracle, wnn32
        coracle.build()
        n_cpu = min(2, images)
        stacks = [np.asarray(tfhe.to_host(h.rgsw.expand())) for h in host[:n_cpu]]
        c0 = time.perf_counter()
        wnn32.he_train(stacks, s, l, a, r, P)
        dt = time.perf_counter() - c0
        out["cpu_baseline"] = {"value": round(n_cpu / dt, 4), "unit": "images/s", "cores": cpu_threads(),
                               "kind": "port", "sample": f"{n_cpu} cfg{cfg} images, oracle/wnn32.he_train "
                                                         f"(C oracle exact ext products, OpenMP)"}
    return out


def bench_cfg4_full(args, torch):
    """BASELINE cfg4 at full size on the stated feasible variant CFG4V:
    16,384 training images (client encryption on the GPU with device-drawn normals,
    streamed into he_train), decrypted counters checked against train_integer, the 2,048
    test images through PD-act inference (predictions == evaluate_dataset), and the fully
    encrypted bleach/popcount/argmax inference on a few test images."""
    from paper_2403_20190_b200 import data, hewnn, infer_pbs, tfhe, wnn
    from paper_2403_20190_b200.params import named_params
    (s, l, a, r, _), _ = data.CONFIG_GEOMETRY[4]
    P = named_params("CFG4V")
    geom = wnn.WisardGeometry(s, l, a, r, P.p)
    n_train, n_test = args.cfg4_train, args.cfg4_test
    ds = data.config_dataset(4, n=n_train, seed=0)
    tds = data.config_dataset(4, split="test", n=n_test, seed=0)
    key = tfhe.SecretKey(P, tfhe.make_rng(KEY_SEED).integers(0, 2, P.n).astype(np.uint32))
    rng = tfhe.make_rng(ENC_SEED)

    def stream():
        for i in range(n_train):
            yield hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits,
                                       device_noise=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    model = hewnn.he_train(stream(), geom, P, batch=args.train_batch)
    e1.record()
    e1.synchronize()
    wall = time.perf_counter() - t0
    dm, cc = hewnn.decrypt_model(model, key)
    ref, rc = wnn.train_integer(ds.bits, ds.labels, geom)
    ok = bool(np.array_equal(dm.counters, ref.counters))
    # class counts are encrypted counters too (decrypt mod p, hw/hewnn.py:323-326); the one
    # ciphertext receives all deposits and its systematic IVP rounding bias
    cc_ok = bool(np.array_equal(cc.counts, rc.counts % P.p))
    cct = tfhe.to_host(model.counts_ct)
    cph = (cct[1].astype(np.int64) - tfhe._key_mul_host(cct[0], key.s).astype(np.int64)) % (1 << 32)
    cerr = np.abs(((cph[:l] + P.delta // 2) % P.delta) - P.delta // 2)
    noise, margin = hewnn.model_noise(model, key)
    # PD-act inference over the whole test set (client decrypts, activates, argmaxes)
    _, pksk = tfhe.keygen(P, KEY_SEED)
    act = wnn.ActivationSpec("bin", 0)
    trng = tfhe.make_rng(ENC_SEED + 7)
    preds, inf_ms = [], 0.0
    for c0 in range(0, n_test, 64):
        ts = [hewnn.encrypt_sample(tds.bits[i], None, key, trng, device_noise=True)
              for i in range(c0, min(n_test, c0 + 64))]
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        packs = hewnn.he_infer_pd_batch(model, ts, pksk)
        g1.record()
        g1.synchronize()
        inf_ms += g0.elapsed_time(g1)
        preds += [hewnn.client_finalize(pk, key, act).prediction for pk in packs]
    plain = wnn.evaluate_dataset(ref, tds.bits, act)
    out = {"workload": f"BASELINE cfg4 geometry at full size: {n_train} train / {n_test} test images",
           "params": f"CFG4V: N=2048 Bg=2^10 l=2 n=750 (cfg4), client RGSW sigma = 2^-32 q, p = {P.p}",
           "why_variant": "BASELINE cfg4 (sigma 2^-25, p = 4096) exceeds Delta/2 = 2^19 after one image at "
                          "q = 2^32 (tools/cfg4_noise.py: 4 images -> 4% counters correct)",
           "train_images_per_s": round(n_train / (e0.elapsed_time(e1) * 1e-3), 2),
           "train_wall_s_incl_client_encryption": round(wall, 1),
           "noise": {"max_log2": round(float(np.log2(max(noise, 1))), 2), "margin_log2": round(float(np.log2(margin)), 2)},
           "check": "decrypted RAM counters == train_integer" if ok else "COUNTER MISMATCH",
           "counters_correct": round(float(np.mean(dm.counters == ref.counters)), 8),
           "class_counts": {"decrypt_ok": cc_ok,
                            "max_error_log2_seen": round(float(np.log2(max(int(cerr.max()), 1))), 2),
                            "note": "one ciphertext takes all 16,384 deposits; the reference's IVP rounding "
                                    "bias (+2^14.7 per deposit, tools/ivp_bias.py) exceeds Delta/2 -- class "
                                    "balancing is unavailable at this size (counters are unaffected)"},
           "infer_pd": {"images_per_s": round(n_test / (inf_ms * 1e-3), 2), "images": n_test,
                        "accuracy": round(float(np.mean(np.array(preds) == tds.labels)), 4),
                        "check": "predictions == evaluate_dataset(bin 0)" if list(plain) == preds
                        else "PREDICTION MISMATCH"}}
    if args.cfg4_pbs_images > 0:
        sbk = infer_pbs.self_bootstrap_keygen(key, KEY_SEED + 11)
        tsm = [hewnn.encrypt_sample(tds.bits[i], None, key, trng) for i in range(args.cfg4_pbs_images)]
        stats: dict = {}
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        pr = infer_pbs.he_infer_bin_batch(model, tsm, sbk, 0, stats=stats)
        g1.record()
        g1.synchronize()
        got = [infer_pbs.decrypt_prediction(x, key) for x in pr]
        want = list(wnn.evaluate_dataset(ref, tds.bits[: args.cfg4_pbs_images], act))
        sec = g0.elapsed_time(g1) * 1e-3
        out["infer_pbs"] = {"images_per_s": round(len(tsm) / sec, 3), "pbs_per_s": round(stats["pbs"] / sec, 1),
                            "pbs_per_image": stats["pbs"] // len(tsm), "images": len(tsm),
                            "self_bsk": "n = N = 2048",
                            "check": "encrypted argmax == evaluate_dataset(bin 0)" if got == want
                            else "PREDICTION MISMATCH"}
    return out


def bench_infer_pbs(args, model, key, ref, tsamples, tbits, torch):
    """OTF-act inference entirely on ciphertexts (paper_2403_20190_b200.infer_pbs):
    VP lookups, bleaching threshold, popcount and argmax on the batched PBS engine,
    self-bootstrapping (n = N) under the training key; the client only decrypts
    the class index.  Checked against wnn.evaluate_dataset(bin thr)."""
    from paper_2403_20190_b200 import infer_pbs, wnn
    thr = args.infer_pbs_thr
    k0 = time.perf_counter()
    sbk = infer_pbs.self_bootstrap_keygen(key, KEY_SEED + 11)
    keygen_s = time.perf_counter() - k0
    infer_pbs.he_infer_bin_batch(model, tsamples[:1], sbk, thr)          # warm-up (LUT tables, workspaces)
    torch.cuda.synchronize()
    stats: dict = {}
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    preds = infer_pbs.he_infer_bin_batch(model, tsamples, sbk, thr, stats=stats)
    g1.record()
    g1.synchronize()
    sec = g0.elapsed_time(g1) * 1e-3
    got = [infer_pbs.decrypt_prediction(p, key) for p in preds]
    want = list(wnn.evaluate_dataset(ref, tbits, wnn.ActivationSpec("bin", thr)))
    n = len(tsamples)
    return {"metric": "encrypted bleaching-threshold inference images/sec", "unit": "images/s",
            "value": round(n / sec, 3), "images": n, "thr": thr,
            "pbs_per_s": round(stats["pbs"] / sec, 1), "pbs_per_image": stats["pbs"] // n,
            "pbs_rounds": stats["rounds"], "self_bsk": f"n = N = {model.params.n} (no key switch)",
            "client_keygen_s": round(keygen_s, 2),
            "note": "timed region includes the VP lookups; PBS/s counts bootstraps only",
            "check": "encrypted argmax == evaluate_dataset(bin thr)" if got == want else "PREDICTION MISMATCH"}


def bench_hwb(args):
    import torch
    import torch.distributed as dist

    from paper_2403_20190_b200 import _lib, tfhe
    from paper_2403_20190_b200.params import named_params

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.set_variant(args.variant)
    _lib.check(_lib.load().hwb_set_fft_mode(args.fft_mode))

    P = named_params("CFG2")
    B = args.batch
    keys, ms, lwe, tv = workload(P, B, rank)
    bsk, ksk = keys.device_keys()
    lwe_d = tfhe.to_device(lwe)
    tv_d = tfhe.to_device(tv)
    ext_d = torch.empty((B, P.n + 1), dtype=torch.int32, device="cuda")
    out_d = torch.empty((B, P.lwe_n + 1), dtype=torch.int32, device="cuda")
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    ks_tc = tfhe._ks_engine(P, ksk, args.ks_engine)
    ks_engine = "tcgen05 kind::i8 (keyswitch_tc_kernel)" if ks_tc else "integer pipe (keyswitch_kernel)"

    def step():
        tfhe.pbs_batch(P, lwe_d, tv_d, bsk, None, out=ext_d, ladder=args.ladder)   # blind rotation + extract
        tfhe.lwe_keyswitch(P, ext_d, ksk, out=out_d, engine=args.ks_engine)   # key switch

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.zero_()                                                 # L2 flush, untimed
        e0, e1, e2 = evs[k]
        e0.record()
        tfhe.pbs_batch(P, lwe_d, tv_d, bsk, None, out=ext_d, ladder=args.ladder)
        e1.record()
        tfhe.lwe_keyswitch(P, ext_d, ksk, out=out_d, engine=args.ks_engine)
        e2.record()
    torch.cuda.synchronize()
    clock_info = clocks.stop()
    if world > 1:
        dist.barrier()
    br_ms = [evs[k][0].elapsed_time(evs[k][1]) for k in range(args.steps)]
    ks_ms = [evs[k][1].elapsed_time(evs[k][2]) for k in range(args.steps)]
    total_ms = sum(br_ms) + sum(ks_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())

    # correctness of the timed outputs (decryption of every ciphertext)
    out_h = tfhe.to_host(out_d)
    dec = tfhe.dec_lwe_batch(out_h, keys.lwe_key)
    ok = bool(np.array_equal(dec, expected(ms, P.p)))

    # end to end through the public API from pinned host memory
    lwe_pin = torch.from_numpy(lwe.view(np.int32)).pin_memory()
    out_pin = torch.empty((B, P.lwe_n + 1), dtype=torch.int32).pin_memory()
    e2e_ms = []
    for k in range(args.steps + 1):
        flush.zero_()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        dev_in = lwe_pin.to("cuda", non_blocking=True)
        res = tfhe.pbs_batch(P, dev_in, tv_d, bsk, ksk, engine=args.ks_engine, ladder=args.ladder)
        out_pin.copy_(res, non_blocking=True)
        e_ev.record()
        e_ev.synchronize()
        if k:                                                         # first = warm-up
            e2e_ms.append(s_ev.elapsed_time(e_ev))
    e2e_ok = bool(np.array_equal(out_pin.numpy().view(np.uint32), out_h))
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)

    # roofline of the dominant kernel (blind rotation) over its event time.
    # NTT ladder: W_mm RNS modmuls per PBS (SURVEY.md §8(d) NTT formulation) vs the
    # measured P_mm.  FFT ladder: W_fp64 FP64 instructions per PBS vs the measured
    # DFMA rate P_fp64 (both counts in DESIGN.md §4-5).
    use_fft = tfhe._use_fft_ladder(bsk, B, args.ladder)
    lv, N, logN = P.gadget.levels, P.n, P.degree_log
    w_cmux = 2 * lv * (N // 2) * logN + 2 * (N // 2) * logN + 4 * lv * N   # 53,248 at cfg2
    w_mm = P.lwe_n * w_cmux
    H, logH = N // 2, logN - 1
    w_fstep = (2 * lv + 4) * (H // 2) * logH * 8 + 2 * lv * 4 * H * 4 + 2 * lv * N + 4 * N   # 243,712 at cfg2
    w_fp64 = P.lwe_n * w_fstep
    br_avg_s = statistics.mean(br_ms) * 1e-3
    if use_fft:
        peak = probe_fp64_peak(torch, _lib, tfhe)
        achieved = w_fp64 * B / br_avg_s
        w_main, unit_main = w_fp64, "G FP64-instr/s"
        roof_kernel = f"{FFT_KERNELS[args.fft_mode]} (FP64 FFT ladder, FFT mode {args.fft_mode})"
        work_txt = f"W_fp64 = {w_fp64} FP64 instructions (n x {w_fstep} per CMUX)"
        peak_src = "measured live: probe_fp64_kernel (8 independent DFMA chains per thread)"
    else:
        peak = probe_modmul_peak(torch, _lib, tfhe)
        achieved = w_mm * B / br_avg_s
        w_main, unit_main = w_mm, "Gmodmul/s"
        roof_kernel = "blind_rotate_kernel<1024,PBS> (two-prime NTT ladder)"
        work_txt = f"W_mm = {w_mm} RNS modmuls (n x 53,248 per CMUX)"
        peak_src = "measured live: probe_modmul_kernel (register-only Shoup, both primes)"
    # key switch: W_ks int32 MACs; on tensor cores 4 byte limbs
    w_ks = P.n * P.gadget_ks.levels * (P.lwe_n + 1)
    ks_avg_s = statistics.mean(ks_ms) * 1e-3
    if ks_tc:
        p_ks, ks_unit, w_ks_eff = probe_i8mma_peak(torch, _lib, tfhe), "int8 MAC/s", 4 * w_ks
    else:
        p_ks, ks_unit, w_ks_eff = None, "int32 MAC/s", w_ks
    # PBS-level roofline: 1 / (W_mm/P_mm + W_ks/P_ks)
    pbs_roof = 1.0 / (w_main / peak + (w_ks_eff / p_ks if p_ks else 0.0))
    # the metric's "% of int roofline": SURVEY §8(d)'s integer-pipe roofline of the NTT
    # formulation (W_mm modmuls per PBS at the measured P_mm, plus the key switch),
    # which the FFT ladder beats by computing the same exact products on the FP64 pipe
    p_mm = peak if not use_fft else probe_modmul_peak(torch, _lib, tfhe)
    int_roof = 1.0 / (w_mm / p_mm + (w_ks_eff / p_ks if p_ks else 0.0))

    value = B * world * args.steps / (max_ms * 1e-3)
    smem_roof = None
    if use_fft:
        # the FFT ladder's binding resource is on-chip: shared-memory bandwidth
        # (128 B/clk/SM).  Algorithmic bytes per ciphertext-step:
        # transposes (2 per transform, write + read), the key slices (TMA write +
        # LDS read), digit extraction and byte digits, accumulator update.
        Hf = N // 2
        if args.fft_mode == 5:
            # lane-paired TMEM ladder: a key / twiddle LDS.128 serves a lane pair (2 of 4
            # wavefronts per warp instruction, tools/lds_bcast_bench.cu), each staged
            # slice 4 ciphertexts (TMA write); decomposition words once per component;
            # compact per-thread twiddles (8 per transform) from shared memory
            smem_step = ((2 * lv + 4) * 2 * 2 * Hf * 16 + 2 * lv * 2 * 2 * Hf * 16 * (1 / 4 + 1 / 2)
                         + (2 * lv + 4) * 8 * 64 * 16 / 2 + 2 * N * 4 * 2 + 2 * N * 4 * 2)
        elif args.fft_mode == 1:
            # TMEM accumulators: each key value read serves 2 ciphertexts, each staged
            # slice 4; digits re-extracted per digit row (rotated + plain reads)
            smem_step = ((2 * lv + 4) * 2 * 2 * Hf * 16 + 2 * lv * 2 * 2 * Hf * 16 * (1 / 4 + 1 / 2)
                         + 2 * lv * N * 4 + 2 * N * 4 * 2)
        else:
            smem_step = ((2 * lv + 4) * 2 * 2 * Hf * 16 + 2 * (2 * lv * 2 * 2 * Hf * 16)
                         + 2 * N * 4 * 2 + 2 * 2 * lv * N + 2 * N * 4 * 2)
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        mhz = (clock_info or {}).get("sm_mhz") or 1965.0
        sm_peak = 128.0 * sms * mhz * 1e6
        sm_ach = smem_step * P.lwe_n * B / br_avg_s
        smem_roof = {"bound": "smem", "achieved": round(sm_ach / 1e12, 2), "peak": round(sm_peak / 1e12, 2),
                     "unit": "TB/s", "frac": round(sm_ach / sm_peak, 4),
                     "bytes_per_step": smem_step,
                     "peak_source": f"128 B/clk/SM x {sms} SMs x {mhz:.0f} MHz (median SM clock under load)",
                     "ncu": "profiles/r02c_ncu_td.txt: l1tex throughput (LSU wavefronts + TMA writes) "
                            "0.74 of peak; the register ladder reached 0.89 (profiles/r01_ncu_fft_ladder_v2.txt)"}
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded LWE encryptions, BASELINE cfg2 shapes)",
        "config": config(P, B, world, {"kernel_variant": args.variant, "ks_engine": ks_engine,
                                       "ladder": "fp64 FFT" if use_fft else "two-prime NTT",
                                       "launch": {"ranks": world, "backend": dist.get_backend() if world > 1
                                                  else None, "nccl_nranks": world if world > 1 else None,
                                                  "requested_gpus": args.gpus}}),
        "e2e": {"value": round(B * world * args.steps / (float(e2e_t.item()) * 1e-3), 2), "unit": UNIT,
                "h2d_bytes_per_step": int(lwe.nbytes), "d2h_bytes_per_step": int(out_h.nbytes),
                "api": "tfhe.pbs_batch from pinned host tensors", "matches_device_run": e2e_ok},
        "roofline": {"bound": "fp64" if use_fft else "int", "kernel": roof_kernel,
                     "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2),
                     "unit": unit_main, "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(B, (P.lwe_n * 2 * lv * 2 * 2 * (N // 2) * 16 if use_fft
                                                else 4 * P.lwe_n * 2 * lv * 2 * 2 * N)
                                               + 4 * (B * (P.lwe_n + 1) + B * (N + 1) + 2 * N),
                                            FFT_KERNELS[args.fft_mode] if use_fft else "ntt"),
                     "work_per_pbs": work_txt, "peak_source": peak_src,
                     "traffic_note": ("DRAM bytes of the ladder's single launch (one batch), ncu --set full "
                                      "--clock-control none, profiles/r02c_ncu_td.txt: the key streams once per "
                                      "batch, the segment accumulators (B x 8 KB) stay in L2 between segments")
                     if use_fft else None,
                     "context": {}}}
    ctx = {"pbs": {"roofline_pbs_per_s": round(pbs_roof, 1),
                             "frac": round(B / (max_ms / args.steps * 1e-3) / pbs_roof, 4),
                             "formula": ("1 / (W/P + 4 W_ks/P_i8)" if ks_tc else "W/P only")
                             + (" with W = W_fp64, P = P_fp64" if use_fft else " with W = W_mm, P = P_mm")},
                     "keyswitch": {"bound": "tensor" if ks_tc else "int", "kernel": ks_engine,
                                   "achieved": round(w_ks_eff * B / ks_avg_s / 1e12, 3),
                                   "peak": round(p_ks / 1e12, 3) if p_ks else None, "unit": "T" + ks_unit,
                                   "frac": round(w_ks_eff * B / ks_avg_s / p_ks, 4) if p_ks else None,
                                   "work_per_pbs": f"{w_ks_eff} MACs",
                                   "peak_source": "measured live: probe_i8mma_kernel (M128 N256 K32 from smem)"
                                   if ks_tc else None},
                     "smem": smem_roof,
                     "int_pipe": {"bound": "int", "roofline_pbs_per_s": round(int_roof, 1),
                                  "frac": round(B / (max_ms / args.steps * 1e-3) / int_roof, 4),
                                  "peak": round(p_mm / 1e9, 2), "unit": "G RNS-modmul/s",
                                  "work_per_pbs": f"W_mm = {w_mm} RNS modmuls (NTT formulation, SURVEY §8(d))",
                                  "formula": "1 / (W_mm/P_mm + 4 W_ks/P_i8)" if ks_tc else "W_mm/P_mm",
                                  "peak_source": "measured live: probe_modmul_kernel (register-only Shoup, both primes)",
                                  "note": ("context only: SURVEY §8(d)'s roofline of the NTT formulation on the "
                                           "integer pipe; the FFT ladder computes the same exact products on the "
                                           "FP64 pipe, whose own fraction (above) is the number of record")}}
    result["roofline"]["context"] = ctx
    result.update({
        "kernel_ms": {"blind_rotate": round(statistics.mean(br_ms), 3),
                      "keyswitch": round(statistics.mean(ks_ms), 3)},
        # the ladder: one launch per batch in FFT mode 5 (>= 4 ciphertexts per SM), else one per
        # 64-step segment; + key-switch digits and GEMM.  (The progress words' memset is a
        # driver memset node, not one of this repo's kernels.)
        "gpu_launches": (((1 if args.fft_mode == 5 and B >= 4 * 148 else -(-P.lwe_n // 64)) if use_fft else 1)
                         + (2 if ks_tc else 1)) * args.steps,
        "clocks": clock_info,
        "check": "all outputs decrypt to the LUT" if ok else "DECRYPTION MISMATCH",
    })
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        sample = args.cpu_sample or max(16, min(256, 2 * threads))
        rate, ref_out = run_cpu_port(P, keys, lwe, tv, sample, threads)
        result["cpu_baseline"] = {
            "value": round(rate, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} cfg2 PBS of the same batch (oracle/c exact schoolbook, "
                      f"OpenMP {threads} threads, {cpu_model()})",
            "bit_exact_vs_gpu": bool(np.array_equal(ref_out, out_h[:sample]))}
    if args.sweep:
        # BASELINE cfg2 batch sweep 1..65536: PBS/s and per-batch latency, device-resident
        sweep = {}
        rng_s = tfhe.make_rng(ENC_SEED + 99)
        for Bs in [int(x) for x in args.sweep.split(",")]:
            ms_s = rng_s.integers(0, P.p, Bs)
            lw = tfhe.to_device(tfhe.enc_lwe_batch(ms_s * P.delta, keys.lwe_key, rng_s))
            tfhe.pbs_batch(P, lw, tv_d, bsk, ksk, engine=args.ks_engine, ladder=args.ladder)   # warm-up
            reps = 3 if Bs <= 4096 else 1
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s0.record()
            for _ in range(reps):
                res = tfhe.pbs_batch(P, lw, tv_d, bsk, ksk, engine=args.ks_engine, ladder=args.ladder)
            s1.record()
            s1.synchronize()
            t_ms = s0.elapsed_time(s1) / reps
            ok_s = bool(np.array_equal(tfhe.dec_lwe_batch(tfhe.to_host(res), keys.lwe_key), expected(ms_s, P.p)))
            sweep[str(Bs)] = {"pbs_per_s": round(Bs / (t_ms * 1e-3), 1), "latency_ms": round(t_ms, 3),
                              "decrypt_ok": ok_s}
            del lw, res
        result["sweep"] = sweep
    if args.other_configs:
        # the other BASELINE PBS parameter sets (cfg1: n=500, l=2, 2^8; cfg4: N=2048,
        # n=750, l=2, 2^10), same batch, device-resident, decryption checked
        other = {}
        peaks = {"fft": probe_fp64_peak(torch, _lib, tfhe), "ntt": probe_modmul_peak(torch, _lib, tfhe)}
        for name in ("CFG1", "CFG4"):
            Po = named_params(name)
            ko, mo, lo, tvo = workload(Po, B, rank)
            bo, kso = ko.device_keys()
            lwo, tvd = tfhe.to_device(lo), tfhe.to_device(tvo)
            res = tfhe.pbs_batch(Po, lwo, tvd, bo, kso, ladder=args.ladder)   # warm-up
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s0.record()
            for _ in range(2):
                res = tfhe.pbs_batch(Po, lwo, tvd, bo, kso, ladder=args.ladder)
            s1.record()
            s1.synchronize()
            t_ms = s0.elapsed_time(s1) / 2
            lvo, No, lgo = Po.gadget.levels, Po.n, Po.degree_log
            fft_o = tfhe._use_fft_ladder(bo, B, args.ladder)
            if fft_o:
                w_o = Po.lwe_n * ((2 * lvo + 4) * (No // 4) * (lgo - 1) * 8 + 2 * lvo * 4 * (No // 2) * 4
                                  + 2 * lvo * No + 4 * No)
            else:
                w_o = Po.lwe_n * (2 * lvo * (No // 2) * lgo + 2 * (No // 2) * lgo + 4 * lvo * No)
            entry = {"pbs_per_s": round(B / (t_ms * 1e-3), 1), "ms_per_batch": round(t_ms, 3),
                     "ladder": "fp64 FFT" if fft_o else "two-prime NTT",
                     "roofline_frac": round(w_o * B / (t_ms * 1e-3) / peaks["fft" if fft_o else "ntt"], 4),
                     "params": f"n={Po.lwe_n} N={No} Bg=2^{Po.gadget.base_log} l={lvo}"}
            if Po.p * 2 <= No:   # PBS decryption is meaningful (>= 2 phase units per message)
                entry["decrypt_ok"] = bool(np.array_equal(tfhe.dec_lwe_batch(tfhe.to_host(res), ko.lwe_key),
                                                          expected(mo, Po.p)))
            other[name.lower()] = entry
            del bo, kso, lwo, res
        result["other_configs"] = other
    if args.train_images > 0:
        result["train"] = bench_train(args, world, rank, torch, dist)
        if args.other_configs:
            # the other BASELINE training workloads (cfg5 RGB 7 classes; cfg4 N = 2048)
            result["train"]["other_configs"] = {f"cfg{c}": train_other(c, n, b, rank, torch)
                                                for c, n, b in ((5, 32, 16), (4, 16, 8))}
        if args.cfg4_full and rank == 0:
            result["train"]["cfg4_full"] = bench_cfg4_full(args, torch)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def bench_reference(args):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return
    from paper_2403_20190_b200.params import named_params
    P = named_params("CFG2")
    threads = cpu_threads()
    sample = args.cpu_sample or max(16, min(256, 2 * threads))
    keys, ms, lwe, tv = workload(P, sample, 0)
    for _ in range(args.warmup):
        run_cpu_port(P, keys, lwe, tv, min(sample, threads), threads)
    rates = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, out = run_cpu_port(P, keys, lwe, tv, sample, threads)
        rates.append(r)
    wall = time.perf_counter() - t0
    from paper_2403_20190_b200 import tfhe
    ok = bool(np.array_equal(tfhe.dec_lwe_batch(out, keys.lwe_key), expected(ms, P.p)))
    value = sample * args.steps / wall
    desc = (f"{sample} cfg2 PBS per step (oracle/c: exact schoolbook port of the reference's "
            f"blind_rotate/extract path + restated KS, OpenMP {threads} threads, {cpu_model()})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(wall / args.steps * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config(P, args.batch, world, {"cpu_sample_per_step": sample}),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "check": "all outputs decrypt to the LUT" if ok else "DECRYPTION MISMATCH",
    }), flush=True)


def _self_launch(args) -> bool:
    """`bench.py --gpus N` outside torchrun: re-exec this script under
    torch.distributed.run with N ranks (one per GPU, NCCL, 127.0.0.1 rendezvous) so
    a direct call really runs on N GPUs.  Returns True when the child ran."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)
    return True


def main():
    args = parse()
    if _self_launch(args):
        return
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_hwb(args)


if __name__ == "__main__":
    main()
