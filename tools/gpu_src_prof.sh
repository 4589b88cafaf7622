# per-source-line ncu captures of the hot kernels (C4 sort / count / join, C3 grouping / probe)
O=gpurun_out/src1
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/lsj_diag.py > $O/lsj_diag.txt 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 1200 $NCU -k regex:"k_lsj_sort|k_est_sample|k_lsj_join|k_split_scatter|k_split_count" -c 10 -o $O/c4 python tools/one_step.py c4 x 1 > $O/c4.log 2>&1
ncu -i $O/c4.ncu-rep --page source --csv --print-source=cuda,sass > $O/c4_source.csv 2>/dev/null
python tools/ncu_sum.py $O/c4.ncu-rep > $O/c4_sum.txt 2>&1
for k in k_lsj_sort k_est_sample k_lsj_join; do
  ncu -i $O/c4.ncu-rep --page source --csv --print-source=cuda --kernel-name regex:$k -c 1 > $O/c4_${k}_cuda.csv 2>/dev/null
  python tools/ncu_lines.py $O/c4_${k}_cuda.csv instr > $O/c4_${k}_lines_instr.txt 2>&1
  python tools/ncu_lines.py $O/c4_${k}_cuda.csv stall > $O/c4_${k}_lines_stall.txt 2>&1
done
timeout 1200 $NCU -k regex:"k_hash_probe_staged|k_bin_scatter_est" -c 2 -o $O/c3 python tools/one_step.py c3 buffered 1 > $O/c3.log 2>&1
for k in k_hash_probe_staged k_bin_scatter_est; do
  ncu -i $O/c3.ncu-rep --page source --csv --print-source=cuda --kernel-name regex:$k -c 1 > $O/c3_${k}_cuda.csv 2>/dev/null
  python tools/ncu_lines.py $O/c3_${k}_cuda.csv instr > $O/c3_${k}_lines_instr.txt 2>&1
  python tools/ncu_lines.py $O/c3_${k}_cuda.csv stall > $O/c3_${k}_lines_stall.txt 2>&1
done
rm -f $O/c4_source.csv
ls -la $O
