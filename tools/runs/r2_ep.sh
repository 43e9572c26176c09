mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_ep2.so $L/libpgrid_ep6.so $L/libpgrid_ep8.so $L/libpgrid.so $L/libpgrid_ep6.so $L/libpgrid_ep8.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|pairs_emit\|value"
