for st in poisson27 poisson7; do python tools/spmv_micro.py --stencil $st 2>&1 | tail -1; CS_LIB=paper_2603_09790_b200/lib/var/notma.so python tools/spmv_micro.py --stencil $st 2>&1 | tail -1; done
CS_SELL_EXPLICIT=1 python tools/spmv_micro.py --stencil poisson27 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -q -x --timeout 500 2>&1 | tail -3
