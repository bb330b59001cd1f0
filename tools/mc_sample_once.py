import sys, torch; sys.path.insert(0, ".")
import __graft_entry__; __graft_entry__.build()
from paper_2407_00047_b200 import RwtEstimator
from workloads.synth import make_config
e = RwtEstimator(make_config("C3"))
for _ in range(3): e.mc_sample(2, 1221)
torch.cuda.synchronize()
