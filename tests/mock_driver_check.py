"""Host-mode shard driver on MOCK devices (no GPU): run in a fresh process
with LP2D_B200_MOCK_DEVICES=N and LP2D_B200_CHUNK_ELEMS=E set (the library
reads them once). Prints one JSON line with the per-LP gather record."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1902_04995_b200 as P  # noqa: E402


def main():
    sizes = np.array([int(x) for x in sys.argv[1].split(",")], np.int32)
    n_gpus = int(sys.argv[2])
    dt = np.float32 if sys.argv[3] == "f32" else np.float64
    pb = P.PackedBatch.generate(sizes, 5).astype(dt)
    r = P.solve_packed(pb, P.BlockConfig(workers=n_gpus))
    print(json.dumps({"status": r.status.tolist(), "x": r.x.tolist(), "shard": r.y.tolist(),
                      "chunk": r.value.tolist(), "wu": r.work_units.tolist(),
                      "offset": pb.offset.tolist()}))


if __name__ == "__main__":
    main()
