import torch, time
x = torch.empty(1024 * 2**20 // 4, dtype=torch.int32).pin_memory()
d = torch.empty_like(x, device="cuda")
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
cs = torch.cuda.Stream()
def copy():
    with torch.cuda.stream(cs):
        d.copy_(x, non_blocking=True)
def comp():
    for _ in range(20): a @ a
def t(f):
    torch.cuda.synchronize(); s = time.perf_counter(); f(); torch.cuda.synchronize(); return (time.perf_counter() - s) * 1e3
copy(); comp(); torch.cuda.synchronize()
print("copy", t(copy), "comp", t(comp), "both", t(lambda: (copy(), comp())))
print("main stream", torch.cuda.current_stream(), "cs", cs)
