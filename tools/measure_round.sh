#!/bin/bash
# Round measurement pass on one B200 (run under gpurun): every bench config, the reference arm,
# the ncu launch list of the cfg2 path (host-driven mode) and --set full captures of K4 (k_chol_d2) and K1.
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/m_smi.txt
python bench.py > gpurun_out/m_cfg2.json 2> gpurun_out/m_cfg2.err
python bench.py --config cfg1 > gpurun_out/m_cfg1.json 2> gpurun_out/m_cfg1.err
python bench.py --config cfg3 > gpurun_out/m_cfg3.json 2> gpurun_out/m_cfg3.err
python bench.py --config cfg4 > gpurun_out/m_cfg4.json 2> gpurun_out/m_cfg4.err
python bench.py --config cfg4 --geno > gpurun_out/m_cfg4g.json 2> gpurun_out/m_cfg4g.err
python bench.py --config cfg5 --no-e2e > gpurun_out/m_cfg5.json 2> gpurun_out/m_cfg5.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/m_launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --control host > gpurun_out/m_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_chol_d2 -s 40 -c 1 -o gpurun_out/m_d2 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --control host > gpurun_out/m_ncu_d2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_aty_fused -s 30 -c 1 -o gpurun_out/m_k1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --control host > gpurun_out/m_ncu_k1.log 2>&1
echo done
