import sys, os
sys.path.insert(0, os.getcwd())
from paper_2101_08734_b200 import clairplan as cp
F, N, b, E = 14_197_122, 1024, 32, 90
sizes = cp.generate_sizes(F, 0.1077, 0.2, 1_500_000.0, 1)
wr = (int(sys.argv[1]), int(sys.argv[2]))
p = cp.Plan(42, F, cp.PartitionSpec(N, b * N, E, True), [120000.0, 900000.0], sizes, worker_range=wr)
p.build()
print(wr, p.stats(), flush=True)
