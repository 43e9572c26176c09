mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_k4m8.so $L/libpgrid_rs3.so $L/libpgrid.so $L/libpgrid_k4m8.so $L/libpgrid_rs3.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|cell_offsets\|radix_scatter\|total\|value"
