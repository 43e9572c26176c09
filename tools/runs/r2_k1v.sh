mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_k1r1.so $L/libpgrid_k1r4.so $L/libpgrid_k1t128r4.so $L/libpgrid.so $L/libpgrid_k1r1.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|boxes_count\|scan_tile_sums\|pair_tile\|total\|value"
