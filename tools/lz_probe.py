"""Time the fast Lanczos estimate alone (device-resident 27-pt problem).

    python tools/lz_probe.py [N] [reps]      (CS_LZ_GONLY=0: the (v, g) variant)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_09790_b200 as cs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = cs.Context(0)
cs.set_default_context(ctx)
p = cs.DeviceProblem.generate("poisson27", n, n, n, ctx=ctx).set_precond("jacobi")
for i in range(reps):
    ctx.synchronize()
    t0 = time.perf_counter()
    est = p.estimate_interval(40, 1234, "fast")
    ctx.synchronize()
    print(f"lanczos {n}^3 gonly={os.environ.get('CS_LZ_GONLY', '1')}: {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"lambda [{est.lambda_min!r}, {est.lambda_max!r}]", flush=True)
p.close()
