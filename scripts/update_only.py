"""Build + insert + delete on C5-shaped inputs, no k-NN (profiling target; dev aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

c = zdgen.CONFIGS["C5"]
pts = torch.from_numpy(zdgen.config_points("C5")).cuda()
batch = torch.from_numpy(zdgen.insert_batch(c["insert_m"], 3, c["insert_seed"])).cuda()
kill = torch.from_numpy(zdgen.delete_ids(c["n"], c["delete_m"], c["delete_seed"])).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    t = zd.zd_build(pts)
    t.zd_insert(batch)
    t.zd_delete(kill)
    torch.cuda.synchronize()
    t.zd_free()
print("ok")
