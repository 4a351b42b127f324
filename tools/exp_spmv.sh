# SpMV kernel comparison on the C2 operator (natural, kNN-locality and ideal blob orders)
for m in nat perm ideal; do for k in ${KERNELS:-local vec bulk}; do
  SPECLUST_SPMV_KERNEL=$k timeout 300 python tools/prof_spmv.py $m 2>&1 | tail -1 | sed "s/^/$k /"
done; done
