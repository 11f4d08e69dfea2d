import sys, numpy as np, torch
sys.path.insert(0, '.')
import gen
from paper_2407_00829_b200 import sable
np.set_printoptions(linewidth=200, precision=3, suppress=True)
def case(h, w, k, seed=0):
    g = np.random.default_rng(seed)
    A = g.integers(1, 5, (h, w)).astype(np.float32)
    I, J = np.nonzero(A)
    s = gen.Synth(name="dbg", nrows=h, ncols=w, dtype=np.float32, delta=50,
                  rpntr=np.array([0, h], np.int32), cpntr=np.array([0, w], np.int32),
                  rects=np.zeros((0, 4), np.int64), I=I.astype(np.int64), J=J.astype(np.int64),
                  V=A[I, J], x=np.ones(w, np.float32), in_rect=np.ones(len(I), bool))
    arrays = {kk: torch.from_numpy(np.ascontiguousarray(v)).cuda() for kk, v in s.vbr_input("rect").items() if isinstance(v, np.ndarray)}
    M = sable.VbrMatrix(arrays, h, w, delta=50)
    X = np.zeros((w, k), np.float32)
    X[:, :] = g.integers(0, 3, (w, k))
    Y = M.spmm(torch.from_numpy(X).cuda()).cpu().numpy()
    R = A @ X
    print(f"h={h} w={w} k={k} info units={M.info['n_units']} max|err|={np.abs(Y-R).max()}")
    if np.abs(Y - R).max() > 0:
        print("Y-R (rows x first 16 rhs):"); print((Y - R)[:, :16])
        print("R:"); print(R[:, :16])
    M.close()
case(8, 8, 16)
case(8, 8, 16, 1)
case(4, 8, 16)
case(16, 8, 16)
case(8, 16, 16)
case(8, 32, 16)
case(8, 40, 16)
case(32, 64, 128)
