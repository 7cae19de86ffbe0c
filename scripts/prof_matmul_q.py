import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
n = 4096
a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
c = torch.empty((n, n), device="cuda")
for _ in range(2):
    q.quantized_matmul_at(a, b, q.QuantSpec(q.FloatFormat(8, 7)), 0, out=c, sync=False)
torch.cuda.synchronize(); print("ok")
