"""One-time sketch timing on a BASELINE config (profiling driver):
    python scripts/sketch_time.py CONFIG BLOCK
prints (host embedding ms, device sketch ms) for three CurState inits."""
import sys, time
sys.path.insert(0, "/root/repo")
import paper_2604_05065_b200 as apc
ctx = apc.Context(0)
p = apc.Problem(int(sys.argv[1]))
A = apc.DeviceMatrix.from_problem(ctx, p)
for i in range(3):
    cur = apc.CurState(A, int(sys.argv[2]), seed=1)
    print("sketch timing", cur.sketch_timing(), flush=True)
    cur.close()
