"""Where csemb_matrix_upload's time goes (config-2 CSR from pinned host memory)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_08360_b200 as pb  # noqa: E402
from paper_1509_08360_b200 import graphs  # noqa: E402

S = graphs.sbm(1_000_000, 100, 15.0, 5.0, seed=2)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
keep = [pin(S.row_offsets), pin(S.col_indices), pin(S.values)]
ro, ci, va = (t.numpy() for t in keep)
n = S.n_rows
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = [t.to("cuda", non_blocking=True) for t in keep]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    Sk = pb.SparseMatrix(n, n, ro, ci, va, check=False)
    t2 = time.perf_counter()
    dm = pb.DeviceMatrix(Sk, "float64")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    dm.close()
    del dev
    print(f"torch H2D of the 3 arrays {1e3*(t1-t0):.2f} ms | SparseMatrix {1e3*(t2-t1):.2f} ms | "
          f"DeviceMatrix upload {1e3*(t3-t2):.2f} ms", flush=True)
