#!/bin/bash
# A/B a kernel switch on the 256^3 bench: one short device-resident bench per
# environment setting, ms per outer iteration and the solve time printed per run.
#   bash tools/ab_env.sh "CS_BOX_WS=0" "CS_BOX_WS=1" ...
for envs in "$@"; do
  env $envs timeout 900 python bench.py --grid ${AB_GRID:-256} --steps ${AB_STEPS:-3} --warmup 3 --no-e2e --no-cpu --no-pcg 2>/dev/null |
    python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['solve_roofline']
print('$envs', 'outer', d['config']['outer_iters'], 'ms/outer %.4f' % s['t_outer_ms'], 'lanczos %.1f ms' % s['t_lanczos_ms'],
      'value %.5f' % d['value'], 'sm_mhz', d['clocks']['sm_mhz'], 'phases', d['phases_ms'])"
done
