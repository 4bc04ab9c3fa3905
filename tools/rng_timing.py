import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1712_02248_b200 as cb
ctx = cb.Context(0)
for rows, cols in ((10000, 36), (5000, 36), (100000, 70)):
    out = torch.empty((rows, cols), device="cuda")
    for _ in range(2): ctx.gaussian_sketch(rows, cols, 3, out)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): ctx.gaussian_sketch(rows, cols, 3, out)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(os.environ.get("CNMF_MT_JUMP_MIN", "default"), rows, cols, f"{dt*1e6:.0f} us (wall, incl. sync)")
