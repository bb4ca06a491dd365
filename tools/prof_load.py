"""ncu driver: the standalone load-vector kernel at one p (1M prisms)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_1191_b200 as pb  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
E = 2 * 128 * 64 * 64
geom = torch.from_numpy(pb.generate_box_mesh(128, 64, 64, 0.1, 42, soa=True)).cuda()
out = torch.empty(E * pb.shape_count(p), dtype=torch.float64, device="cuda")
f = torch.ones(E, dtype=torch.float64, device="cuda")
with pb.Integrator(p) as it:
    for _ in range(3):
        it.load_vectors_device(E, geom, out, f=f)
    it.check()
print("ok")
