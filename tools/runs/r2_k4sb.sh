mkdir -p gpurun_out
L=paper_2403_10647_b200/_lib
LIBS="$L/libpgrid.so $L/libpgrid_k4sb.so $L/libpgrid.so $L/libpgrid_k4sb.so" bash tools/ab_libs.sh
grep -v '^"parity\|^  ' gpurun_out/ab.log | grep "==\|cell_offsets\|key_tile\|total\|value"
grep '"parity"' gpurun_out/ab.log | sort | uniq -c
