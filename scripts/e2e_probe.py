import sys, time, os
sys.path.insert(0, os.getcwd())
import bench
from paper_1709_09479_b200 import dcsc
cfg = bench.CONFIGS["c1"]
x, d = bench.make_data(cfg, 0, cfg["N"])
sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=bench.SEED, tol=1e-300)
ctx = dcsc.Context(cfg["N"], (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"])
ctx.set_signals(x); ctx.set_dictionary(d)
for _ in range(3):
    ctx.set_coding_state(None, None); ctx.coding()
ctx.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); ctx.set_signals(x); ctx.synchronize(); t1 = time.perf_counter()
    ctx.set_coding_state(None, None); ctx.synchronize(); t2 = time.perf_counter()
    st = ctx.coding(); ctx.synchronize(); t3 = time.perf_counter()
    print(f"set_signals {1e3*(t1-t0):.2f} ms  reset {1e3*(t2-t1):.2f} ms  coding {1e3*(t3-t2):.2f} ms", flush=True)
