# per-source-line instruction / stall totals of the dominant kernels (ncu --set full source page)
O=gpurun_out/lines
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_hash_probe_staged|k_bin_scatter_est" -c 2 -o $O/c3 python tools/one_step.py c3 buffered 1 > $O/c3.log 2>&1
ncu -i $O/c3.ncu-rep --page source --csv --print-source=cuda,sass > $O/c3_src.csv 2>$O/c3_src.err
python tools/ncu_lines.py $O/c3_src.csv instr > $O/c3_lines_instr.txt 2>&1
python tools/ncu_lines.py $O/c3_src.csv stall > $O/c3_lines_stall.txt 2>&1
timeout 1200 $NCU -k regex:"k_lsj_sort|k_split_scatter|k_split_count" -c 4 -o $O/c4 python tools/one_step.py c4 x 1 > $O/c4.log 2>&1
ncu -i $O/c4.ncu-rep --page source --csv --print-source=cuda,sass > $O/c4_src.csv 2>$O/c4_src.err
python tools/ncu_lines.py $O/c4_src.csv instr > $O/c4_lines_instr.txt 2>&1
python tools/ncu_lines.py $O/c4_src.csv stall > $O/c4_lines_stall.txt 2>&1
rm -f $O/c3_src.csv $O/c4_src.csv
du -sh $O
