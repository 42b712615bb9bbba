"""Sharded C4 steps under torch.distributed.run (bench.run_sharded_c4 at the job's world size)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

d = bench.Dist()
for B, k in ((1, 300), (256, 30)):
    r = bench.run_sharded_c4(d, 1_000_000, B, k, 5, device=d.local)
    if d.rank == 0:
        print(json.dumps(r))
d.td.destroy_process_group()
