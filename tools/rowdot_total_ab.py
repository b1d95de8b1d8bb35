import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2202_13007_b200 import device as dev
n = 65536
A, _ = bench._shard_compress("smooth", 0, n, n, 11)
B, _ = bench._shard_compress("smooth", 0, n, n, 12)
def two():
    r = dev.rowdot(A, B); dev.sum_ascending(r)
for i in range(2):
    print(json.dumps({"fused": bench._time_dist(lambda: dev.frobenius(A, B), 3, 1), "two_calls": bench._time_dist(two, 3, 1),
                      "rowdot_only": bench._time_dist(lambda: dev.rowdot(A, B), 3, 1)}))
