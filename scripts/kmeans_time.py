import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_17415_b200.partition import train_partition
rng = np.random.default_rng(0)
x = rng.standard_normal((411644, 96)); x /= np.linalg.norm(x, axis=1)[:, None]
torch.cuda.synchronize(); t = time.perf_counter()
p = train_partition(x, 4096, seed=0, max_iters=25, device="cuda")
torch.cuda.synchronize(); print("kmeans 411k x 4096", time.perf_counter() - t, "s")
