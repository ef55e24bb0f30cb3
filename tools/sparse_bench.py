import sys, json, torch
sys.path.insert(0, '.')
import bench, paper_1802_09113_b200 as snx
print(json.dumps(bench.sparse_rate(snx, torch)))
