import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1205_3830_b200 as rid
A = rid.generate(1, 1024, 512, 16, 0.0)
for _ in range(3): rid.decompose(A, 16, 24, 1)
torch.cuda.synchronize()
