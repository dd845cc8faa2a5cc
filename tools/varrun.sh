for f in paper_2603_09790_b200/lib/var/*.so; do CS_LIB=$f python tools/spmv_micro.py 2>&1 | tail -1; done
CS_LIB=paper_2603_09790_b200/lib/var/CS_PACK_MINB-1.so python tools/spmv_micro.py --stencil poisson7 | tail -1
