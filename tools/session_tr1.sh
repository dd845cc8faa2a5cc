set -u
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_solver.py -q -x -k "fast_mode_parity or golden_counts or device_resident" > $out/t1_tests.log 2>&1; echo "tests rc=$?" >> $out/t1_status.txt
timeout 600 python bench.py --grid 256 --steps 3 --warmup 3 --no-e2e --no-cpu --no-pcg --variant 128 > $out/t1_b256_tr.jsonl 2> $out/t1_b256_tr.err; echo "b256tr rc=$?" >> $out/t1_status.txt
timeout 600 python bench.py --grid 256 --steps 3 --warmup 3 --no-e2e --no-cpu --no-pcg --variant 0 > $out/t1_b256_0.jsonl 2> $out/t1_b256_0.err; echo "b256 rc=$?" >> $out/t1_status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/t1_launches_tr.csv python bench.py --grid 256 --steps 1 --warmup 0 --no-e2e --no-cpu --no-pcg --variant 128 > $out/t1_ncu.log 2>&1; echo "ncu rc=$?" >> $out/t1_status.txt
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-pcg --variant 128 > $out/t1_b512_tr.jsonl 2> $out/t1_b512_tr.err; echo "b512tr rc=$?" >> $out/t1_status.txt
