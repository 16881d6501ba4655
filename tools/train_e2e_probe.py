"""Where does he_train's end-to-end time go?  Times, for cfg3 images encrypted on
the GPU: (1) the pinned H2D of all RGSW stacks alone, (2) he_train on
device-resident stacks, (3) he_train from pinned host stacks (the bench's e2e)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import data, hewnn, tfhe, wnn  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e), (time.perf_counter() - t0) * 1e3


def main(images=128, batch=32):
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[3]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    key, _ = tfhe.keygen(P, 1)
    ds = data.config_dataset(3, n=images)
    rng = tfhe.make_rng(2)
    dev = [hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits, device=True)
           for i in range(images)]
    host = [hewnn.EncryptedSample.from_stack(P, d.rgsw.cpu().pin_memory(), d.s, d.n_label_bits) for d in dev]
    hewnn.he_train(dev[:batch], geom, P, batch=batch)
    hewnn.he_train(host[:batch], geom, P, batch=batch)
    nbytes = sum(h.rgsw.numel() * 4 for h in host)
    ms, _ = timed(lambda: [h.rgsw.to("cuda", non_blocking=True) for h in host])
    print(f"H2D only: {ms:.1f} ms ({nbytes / ms / 1e6:.1f} GB/s)")
    ms, wall = timed(lambda: hewnn.he_train(dev, geom, P, batch=batch))
    print(f"he_train device-resident: {ms:.1f} ms (host {wall:.1f} ms), {images / ms * 1e3:.0f} img/s")
    ms, wall = timed(lambda: hewnn.he_train(host, geom, P, batch=batch))
    print(f"he_train pinned host: {ms:.1f} ms (host {wall:.1f} ms), {images / ms * 1e3:.0f} img/s")
    hewnn._TRACE = []
    base = hewnn._ev()
    t_host = []
    t0 = time.perf_counter()
    hewnn.he_train(host, geom, P, batch=batch)
    torch.cuda.synchronize()
    for label, ev in hewnn._TRACE:
        print(f"  {label:11s} {base.elapsed_time(ev):8.1f} ms")
    hewnn._TRACE = None




def timeline(images=128, batch=32):
    """torch.profiler (CUPTI) timeline of the pinned-host he_train: busy time of
    H2D copies, of kernels, and of their overlap."""
    from torch.profiler import ProfilerActivity, profile
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[3]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    key, _ = tfhe.keygen(P, 1)
    ds = data.config_dataset(3, n=images)
    rng = tfhe.make_rng(2)
    host = [hewnn.EncryptedSample.from_stack(P, hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng,
                                                          label_bits=geom.label_bits).rgsw.cpu().pin_memory(),
                                  s, geom.label_bits) for i in range(images)]
    hewnn.he_train(host[:batch], geom, P, batch=batch)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        hewnn.he_train(host, geom, P, batch=batch)
        torch.cuda.synchronize()
    copies, kernels = [], []
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        iv = (ev.time_range.start, ev.time_range.end)
        (copies if "Memcpy" in ev.name or "memcpy" in ev.name else kernels).append(iv)

    def union(ivs):
        ivs = sorted(ivs)
        tot, cur = 0, None
        for a0, b0 in ivs:
            if cur is None or a0 > cur[1]:
                if cur:
                    tot += cur[1] - cur[0]
                cur = [a0, b0]
            else:
                cur[1] = max(cur[1], b0)
        return tot + (cur[1] - cur[0] if cur else 0)
    span = max(b for _, b in copies + kernels) - min(a for a, _ in copies + kernels)
    uc, uk, ua = union(copies), union(kernels), union(copies + kernels)
    print(f"span {span / 1e3:.1f} ms: copies busy {uc / 1e3:.1f} ms, kernels busy {uk / 1e3:.1f} ms, "
          f"overlap {(uc + uk - ua) / 1e3:.1f} ms")
    t0 = min(a for a, _ in copies + kernels)

    def segments(ivs, gap=200):
        out = []
        for a0, b0 in sorted(ivs):
            if out and a0 - out[-1][1] <= gap:
                out[-1][1] = max(out[-1][1], b0)
            else:
                out.append([a0, b0])
        return out
    for name, ivs in (("copies", copies), ("kernels", kernels)):
        segs = segments(ivs)
        print(name, " ".join(f"[{(a0 - t0) / 1e3:.0f},{(b0 - t0) / 1e3:.0f}]" for a0, b0 in segs[:16]))


if __name__ == "__main__":
    if sys.argv[1:2] == ["timeline"]:
        timeline(*[int(x) for x in sys.argv[2:]])
    else:
        main(*[int(x) for x in sys.argv[1:]])
