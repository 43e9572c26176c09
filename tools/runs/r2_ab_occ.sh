# scatter occupancy variants: ktimes + bench per library (tools/ab_libs.sh)
mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_i12.so $L/libpgrid_t512i8c3.so $L/libpgrid_t512i8.so $L/libpgrid_g32.so $L/libpgrid_g8.so $L/libpgrid.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|radix_scatter\|k_tile_counts\|pairs_emit\|cell_offsets\|key_tile\|total\|value"
