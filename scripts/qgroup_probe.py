import sys, torch, numpy as np
sys.path.insert(0, '.')
import bench
from paper_2510_21270_b200 import ops
bench.HQ, bench.HKV = 32, 8
q, k, v = bench.make_inputs(torch, 131072, 0, 4, [0], 'cuda')
perm, inv = ops.build_query_permutation(q, k, 128, 256)
torch.cuda.synchronize()
# a gaussian case
q2 = torch.randn(4, 131072, 128, device='cuda').to(torch.bfloat16); k2 = torch.randn(1, 131072, 128, device='cuda').to(torch.bfloat16)
perm, inv = ops.build_query_permutation(q2, k2, 128, 256)
torch.cuda.synchronize()
