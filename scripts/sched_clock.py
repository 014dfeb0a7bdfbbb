import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W
n = int(sys.argv[1])
keys, _ = W.generate("uniform", n)
src = torch.from_numpy(keys).cuda()
s = T.Sorter(seed=1)
for _ in range(4):
    d = src.clone(); torch.cuda.synchronize(); s.sort(d)
torch.cuda.synchronize()
