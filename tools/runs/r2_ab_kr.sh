mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_kr.so $L/libpgrid_kr3.so $L/libpgrid_krvl.so $L/libpgrid_krvl3.so $L/libpgrid_vr.so $L/libpgrid.so $L/libpgrid_kr.so $L/libpgrid_kr3.so $L/libpgrid_krvl3.so" bash tools/ab_libs.sh
grep -v '^  ' gpurun_out/ab.log | grep "==\|radix_scatter\|value\|parity"
for v in kr3 krvl3; do
  PGRID_LIB=$PWD/$L/libpgrid_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/ab_tests_$v.txt 2>&1
  echo "$v rc=$?"; tail -n 2 gpurun_out/ab_tests_$v.txt
done
