import torch
G, cap, M, F = 128, 512, 2048, 8192
x = torch.randn(G, cap, M, device="cuda").to(torch.bfloat16)
w = torch.randn(G, F, M, device="cuda", dtype=torch.bfloat16).transpose(1, 2)
h = torch.empty(G, cap, F, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(G, M, F, device="cuda", dtype=torch.bfloat16).transpose(1, 2)
y = torch.empty(G, cap, M, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    torch.bmm(x, w, out=h)
    torch.bmm(h, w2, out=y)
torch.cuda.synchronize()
