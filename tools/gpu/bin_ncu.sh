# binned parallel kernel (rowquad_kernel<solve, bin>): compute floor of the walk (probe build
# without random gathers, CSR order) and ncu captures at two window sizes
O=gpurun_out
L=$PWD/paper_0810_1119_b200/lib
echo "coalesced probe (no random twin gather, CSR order):" > $O/bin_ncu.txt
GABP_ROW_NO_BIN=1 GABP_LIB=$L/libgabp_b200_coal.so python tools/par_probe.py --config 1 --modes rows --solve 0 >> $O/bin_ncu.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
for w in 8 32; do
GABP_BIN_WINDOW_MB=$w python tools/par_probe.py --config 1 --modes rows --solve 0 --sweeps 6 > $O/plain_r.log 2>&1 && \
GABP_BIN_WINDOW_MB=$w $NCU -k regex:rowquad_kernel -s 5 -c 1 -o $O/r02_rowquad_bin_w$w python tools/par_probe.py --config 1 --modes rows --solve 0 --sweeps 6 > $O/ncu_r$w.log 2>&1
done
ls -la $O
