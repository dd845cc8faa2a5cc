#!/bin/bash
# One gpurun session: tag + list of steps, each step's output under gpurun_out/<tag>_<step>.*
#   gpurun -- bash tools/gpu_session.sh <tag> <step> [<step> ...]
# steps: info | tests | tests_fast | precond | band256 | band512 | bench | bench256 | ncu_list |
#        ncu_box | sanitize | smoke | multi2 | bench2 | bench4
set -u
tag=$1; shift
out=gpurun_out
mkdir -p $out
cd "${GRAFT_REPO_ROOT:-.}"
for step in "$@"; do
  echo "== $step $(date +%T)" >> $out/${tag}_status.txt
  case $step in
    info)
      { free -g; nproc; lscpu | head -20; nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,memory.total --format=csv; } > $out/${tag}_info.txt 2>&1 ;;
    tests)
      timeout 1800 python -m pytest tests -m gpu -x -q > $out/${tag}_tests.log 2>&1 ;;
    tests_fast)
      timeout 1500 python -m pytest tests -m "gpu and not slow" -q > $out/${tag}_tests.log 2>&1 ;;
    precond)
      timeout 600 python -m pytest tests/test_gpu_precond.py -q > $out/${tag}_precond.log 2>&1 ;;
    band256)
      timeout 1200 python tools/count_band.py --tree-band --cases p27:256:8 --out $out/${tag}_band.json > $out/${tag}_band.log 2>&1 ;;
    band512)
      timeout 1800 python tools/count_band.py --tree-band --cases p27:512:8 --out $out/${tag}_band512.json > $out/${tag}_band512.log 2>&1 ;;
    bandpz)
      timeout 1500 python tools/count_band.py --skip-ref --variants 0,1,32,33 --cases p27:96:8,p27:128:8,p27:128:4,p7:256:4,p27:256:8,p27:512:8 --out $out/${tag}_bandpz.json > $out/${tag}_bandpz.log 2>&1 ;;
    tests_quick)
      timeout 1200 python -m pytest tests/test_gpu_box.py tests/test_gpu_solver.py tests/test_gpu_kernels.py -q -x -m "gpu and not slow" > $out/${tag}_tests_quick.log 2>&1 ;;
    ncu_boxlz)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sell_box_kernel<.int.7" -s 20 -c 1 \
        -o $out/${tag}_box python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg > $out/${tag}_ncu_box.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"lz2_resid_proj_kernel<.int.24" -s 2 -c 1 \
        -o $out/${tag}_lz python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg > $out/${tag}_ncu_lz.log 2>&1 ;;
    ncu_sep)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"sell_boxsep_kernel<.int.7" -s 20 -c 1 \
        -o $out/${tag}_sep python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg > $out/${tag}_ncu_sep.log 2>&1 ;;
    abws)
      timeout 1500 bash tools/ab_env.sh "CS_BOX_WS=0" "CS_BOX_WS=1" "CS_BOX_WS=0" "CS_BOX_WS=1" > $out/${tag}_abws.txt 2>&1 ;;
    abrz)
      for v in 512 0 512 0; do
        timeout 600 python bench.py --grid 256 --steps 3 --warmup 3 --no-e2e --no-cpu --no-pcg --variant $v 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['solve_roofline']
print('variant $v', 'outer', d['config']['outer_iters'], 'ms/outer %.4f' % s['t_outer_ms'], 'lz %.1f' % s['t_lanczos_ms'], 'value %.5f' % d['value'], 'mhz', d['clocks']['sm_mhz'], d['phases_ms'])"
      done > $out/${tag}_abrz.txt 2>&1 ;;
    ab4xr)
      for g in 256 512; do for v in 0 1 0 1; do
        CS_P2P_ALLREDUCE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
          --master-port $((29700 + v)) bench.py --gpus 4 --grid $g --no-cpu --no-e2e --no-pcg --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['solve_roofline']
print('grid $g xred $v', 'outer', d['config']['outer_iters'], 'ms/outer %.4f' % s['t_outer_ms'], 'value %.5f' % d['value'], 'mhz', d['clocks']['sm_mhz'], d['phases_ms'])"
      done; done > $out/${tag}_ab4xr.txt 2>&1 ;;
    trband)
      timeout 2400 python tools/count_band.py --ref-only --variants 0,256 --cases p27:96:8,p27:128:8,p27:128:4,p7:256:4 --out $out/${tag}_trband.json > $out/${tag}_trband.log 2>&1
      timeout 1800 python tools/count_band.py --skip-ref --variants 0,256 --cases p27:256:8,p27:512:8 --out $out/${tag}_trband.json >> $out/${tag}_trband.log 2>&1 ;;
    e2etrace)
      CS_TRACE=1 timeout 1200 python tools/e2e_trace.py 512 > $out/${tag}_e2etrace.log 2>&1 ;;
    ncu_pz)
      timeout 1200 ncu --set full --clock-control none --import-source on \
        -k regex:"pack_kernel|update_kernel|sell_box_kernel" -s 40 -c 3 -o $out/${tag}_pz \
        python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg > $out/${tag}_ncu_pz.log 2>&1 ;;
    ncu_hot)
      for spec in "box:sell_box_kernel:70:2" "upd:update_kernel:6:1" "pack:pack_kernel:6:1" "lz:cgs_kernel|proj_kernel:70:2"; do
        IFS=: read nm rx sk cn <<< "$spec"
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $sk -c $cn \
          -o $out/${tag}_$nm python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg \
          > $out/${tag}_ncu_$nm.log 2>&1
      done ;;
    updsweep)
      timeout 900 bash tools/upd_sweep.sh > $out/${tag}_updsweep.txt 2>&1 ;;
    lzprobe)
      { python tools/lz_probe.py 256 3; CS_LZ_GONLY=0 python tools/lz_probe.py 256 3;
        python tools/lz_probe.py 512 2; CS_LZ_GONLY=0 python tools/lz_probe.py 512 2;
        timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file $out/${tag}_lz_launches.csv python tools/lz_probe.py 256 1;
        CS_LZ_GONLY=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file $out/${tag}_lz_launches_vg.csv python tools/lz_probe.py 256 1; } > $out/${tag}_lzprobe.txt 2>&1 ;;
    boxsweep)
      timeout 900 bash tools/box_sweep.sh > $out/${tag}_boxsweep.txt 2>&1 ;;
    bench)
      timeout 1500 python bench.py > $out/${tag}_bench.jsonl 2> $out/${tag}_bench.err ;;
    bench256)
      timeout 900 python bench.py --grid 256 > $out/${tag}_bench256.jsonl 2> $out/${tag}_bench256.err ;;
    ncu_list)
      timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $out/${tag}_launches.csv python bench.py --grid 256 --steps 1 --warmup 0 \
        --no-e2e --no-cpu --no-pcg > $out/${tag}_ncu_list.log 2>&1 ;;
    ncu_box)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sell_box_kernel \
        -s 20 -c 1 -o $out/${tag}_box python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e \
        --no-cpu --no-pcg > $out/${tag}_ncu_box.log 2>&1 ;;
    sanitize)
      for tool in memcheck synccheck racecheck; do
        timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_case.py \
          $([ $tool = racecheck ] && echo --quick) > $out/${tag}_sanitize_$tool.log 2>&1
      done ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1 ;;
    multi2)
      timeout 1200 python -m pytest tests/test_gpu_multi.py -q > $out/${tag}_multi.log 2>&1 ;;
    bench2)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29611 bench.py --gpus 2 > $out/${tag}_bench2.jsonl 2> $out/${tag}_bench2.err ;;
    bench4)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29613 bench.py --gpus 4 > $out/${tag}_bench4.jsonl 2> $out/${tag}_bench4.err ;;
    bench4w)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29615 bench.py --gpus 4 --grid 256 --scaling weak --no-cpu > $out/${tag}_bench4w.jsonl 2> $out/${tag}_bench4w.err ;;
    bench2s256)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29617 bench.py --gpus 2 --grid 256 --no-cpu > $out/${tag}_bench2s256.jsonl 2> $out/${tag}_bench2s256.err ;;
    bench4s256)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29619 bench.py --gpus 4 --grid 256 --no-cpu > $out/${tag}_bench4s256.jsonl 2> $out/${tag}_bench4s256.err ;;
    *) echo "unknown step $step" >> $out/${tag}_status.txt ;;
  esac
  echo "   rc=$? $(date +%T)" >> $out/${tag}_status.txt
done
