import torch
E, M, D, F = 16, 2048, 4096, 14336
x = torch.randn(E, M, D, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(E, D, 2 * F, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    torch.bmm(x, w1)
torch.cuda.synchronize()
