mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_tc1.so $L/libpgrid_tc2.so $L/libpgrid.so $L/libpgrid_tc1.so $L/libpgrid_tc2.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|k_tile_counts\|total\|value"
