"""HBM bandwidth by direction on this B200: pure write (fill), pure read
(sum), 1:1 copy — is a write-heavy kernel capped below the copy peak?"""
import torch
n = 1 << 30   # 2 GB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.normal_()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
w = t(lambda: b.fill_(1.0)); print(f"write-only  {2*n/w/1e12:.2f} TB/s")
r = t(lambda: a.sum(dtype=torch.float32)); print(f"read-only   {2*n/r/1e12:.2f} TB/s")
c = t(lambda: b.copy_(a)); print(f"copy (r+w)  {4*n/c/1e12:.2f} TB/s")
