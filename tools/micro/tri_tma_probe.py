import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def k(desc, out_ptr):
    x = desc.load([0, 0])
    offs = tl.arange(0, 32)[:, None] * 32 + tl.arange(0, 32)[None, :]
    tl.store(out_ptr + offs, x)

a = torch.arange(64 * 96, dtype=torch.float32, device="cuda").reshape(64, 96)
out = torch.empty(32 * 32, device="cuda")
desc = TensorDescriptor.from_tensor(a, [32, 32])
h = k[(1,)](desc, out)
torch.cuda.synchronize()
print("ok", torch.equal(out.view(32, 32), a[:32, :32]))
ptx = h.asm["ptx"]
for ln in ptx.splitlines():
    if "tensor" in ln or "mbarrier" in ln or "fence" in ln:
        print(ln.strip())
print("=====PTX")
print(ptx[:6000])
