"""Where the end-to-end time goes: device-resident solve vs the host API
(fresh numpy outputs) vs se_solve into pinned host buffers."""
import ctypes
import os
import sys
import time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch
from paper_2101_07088_b200 import workloads as W, _lib
from paper_2101_07088_b200.slab import SlabSolver

s, p = W.build("c4")
n = s.n
solver = SlabSolver(s, p)
pin_pos = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
pin_pos.copy_(torch.from_numpy(s.positions))
pin_phi = torch.empty(n, dtype=torch.float64, pin_memory=True)
pin_E = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
pos_h = pin_pos.numpy()
for _ in range(3):
    solver.solve(positions=pos_h)

def timeit(f, k=5):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))

d_pos = torch.from_numpy(s.positions).cuda()
d_phi = torch.empty(n, dtype=torch.float64, device="cuda")
d_E = torch.empty((n, 3), dtype=torch.float64, device="cuda")
print("device solve     %.2f ms" % timeit(lambda: solver.solve_device(d_pos.data_ptr(), d_phi.data_ptr(), d_E.data_ptr(), n)))
print("host API (fresh) %.2f ms" % timeit(lambda: solver.solve(positions=pos_h)))
U = ctypes.c_double(); diag = _lib.SeDiag()
flags = _lib.NEED_ENERGY | _lib.NEED_FORCES | _lib.NEED_POTENTIAL | _lib.CORRECTION
def pinned():
    dp = ctypes.POINTER(ctypes.c_double)
    cast = lambda t: ctypes.cast(ctypes.c_void_p(t.data_ptr()), dp)
    _lib.check(solver._lib.se_solve(solver._plan, cast(pin_pos), n, flags, cast(pin_phi),
                                    cast(pin_E), ctypes.byref(U), ctypes.byref(diag)))
print("se_solve pinned  %.2f ms" % timeit(pinned))
def fresh_alloc():
    a = np.empty(n); b = np.zeros((n, 3)); a[:] = 1; b[:] = 1
print("numpy alloc+touch %.2f ms" % timeit(fresh_alloc))

# the bench's e2e loop: events around solve(), previous result kept alive
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
res = solver.solve(positions=pos_h)
for use_flush in (False, True):
    ts = []
    for _ in range(6):
        if use_flush:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t = time.perf_counter()
        res = solver.solve(positions=pos_h)
        e1.record(stream); e1.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t)))
    print("bench-style flush=%s events/wall" % use_flush, [("%.1f/%.1f" % x) for x in ts])
