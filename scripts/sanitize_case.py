"""Small end-to-end exercise of every kernel path for compute-sanitizer (dev aid):
build (2D/3D, duplicates), all-points k-NN for k in {1, 10, 32} with both k-NN
passes forced, external queries, insert, delete, export."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_04182_b200 as zd  # noqa: E402
import zdgen  # noqa: E402

for dim, dist in ((2, "uniform"), (3, "plummer"), (3, "dup")):
    pts = torch.from_numpy(zdgen.points(dist, 5000, dim, seed=5)).cuda()
    t = zd.zd_build(pts)
    for mode in ("auto", "all"):
        os.environ["ZD_KNN_DEFER"] = mode
        for k in (1, 10, 32):
            t.zd_knn(k)
    q = torch.from_numpy(zdgen.uniform(700, dim, seed=6)).cuda()
    t.zd_knn(10, queries=q)
    t.zd_insert(torch.from_numpy(zdgen.uniform(900, dim, seed=7)).cuda())
    t.zd_delete(torch.from_numpy(np.arange(0, 5000, 3, dtype=np.int32)).cuda())
    t.zd_knn(10)
    t.zd_export()
    torch.cuda.synchronize()
    t.zd_free()
print("sanitize case ok")
