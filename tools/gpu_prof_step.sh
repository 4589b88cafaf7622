# ncu --set full of kernel $1 in one bench step of config $2 (tools/one_step.py), tag $3
K=$1; C=$2; T=$3
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/prof/$T python tools/one_step.py $C > gpurun_out/prof/$T.log 2>&1
python tools/ncu_sum.py gpurun_out/prof/$T.ncu-rep > gpurun_out/prof/${T}_sum.txt 2>&1
python tools/ncu_src.py gpurun_out/prof/$T.ncu-rep "$K" 50 > gpurun_out/prof/${T}_src.txt 2>&1
