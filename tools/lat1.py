import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1306_4743_b200 as eik
r, n, dt = 16, 15, torch.float32
M = (n + 1) ** 3
F = torch.ones(M, dtype=dt, device="cuda")
m = torch.zeros(M, dtype=torch.uint8, device="cuda"); m[0] = 1
q = torch.zeros(M, dtype=dt, device="cuda")
s = eik.Solver(loop_mode=1)
for _ in range(3):
    s.solve(F, m, q, cell_size=r, n=n)
print("ok")
