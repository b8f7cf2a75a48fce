#!/bin/bash
# Round measurement pass on one B200 (run under gpurun): the GPU test suite, every bench config, the
# reference arm, the ncu launch lists (cfg2 path and cfg5, host-driven mode: ncu cannot profile the
# kernel nodes of graphs with conditional nodes) and `--set full` captures of the main kernels.
# Everything lands in gpurun_out/r2/; the summaries are copied to profiles/ afterwards.
set -x
cd $GRAFT_REPO_ROOT
O=${MEASURE_OUT:-gpurun_out/r2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
lscpu > $O/lscpu.txt; nproc >> $O/lscpu.txt; free -g >> $O/lscpu.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; echo "gpu tests rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 rc=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_cfg5.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?" >> $O/status.txt
done
timeout 900 python bench.py --config cfg4 --geno --steps 20 --warmup 5 > $O/bench_cfg4_geno.json 2> $O/bench_cfg4g.err; echo "cfg4g rc=$?" >> $O/status.txt
timeout 900 python bench.py --sweep > $O/bench_sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?" >> $O/status.txt
timeout 900 python bench.py --select --cv 5 --steps 5 --warmup 3 > $O/bench_select.json 2> $O/select.err; echo "select rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg2 --shard --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg2_shard.json 2> $O/shard.err; echo "shard rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg2 --shard --shard-comm nccl --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg2_shard_nccl.json 2> $O/shard_nccl.err; echo "shard nccl rc=$?" >> $O/status.txt
(cd tools/probes && bash build.sh > /dev/null 2>&1); timeout 300 tools/probes/read_probe > $O/read_probe.jsonl 2>&1; echo "read probe rc=$?" >> $O/status.txt
timeout 600 python tools/kprof.py --newton 20,100,250,435,700,1165,2000,5000,10193 > $O/kprof_newton.txt 2>&1
# launch lists (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_list2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_list5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_list1.log 2>&1
# --set full captures, summarised on the box (details + raw pages as CSV); the reports themselves are
# deleted (gpurun copies back at most 64 MiB)
summ() { ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null; ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null; ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_sass.csv 2>/dev/null; gzip -f $O/$1_sass.csv; rm -f $O/$1.ncu-rep; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_aty_fused -s 10 -c 1 -o $O/k1_n1e7 python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_k1.log 2>&1
summ k1_n1e7
# the REUSE instantiation's launch served from the kept A^T b (R40): launch 0 is create's lambda_max pass, launch 1 the cold solve's first trial
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_aty_fused -s 1 -c 1 -o $O/k1c_n1e7 python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu --no-e2e --control host > $O/ncu_k1c.log 2>&1
summ k1c_n1e7
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --opt reuse_atb=0 > $O/bench_cfg5_noreuse.json 2> $O/bench_cfg5_noreuse.err; echo "cfg5 noreuse rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e --opt reuse_atb=0 > $O/bench_cfg3_noreuse.json 2> $O/bench_cfg3_noreuse.err; echo "cfg3 noreuse rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu --no-e2e --opt reuse_atb=0 > $O/bench_cfg4_noreuse.json 2> $O/bench_cfg4_noreuse.err; echo "cfg4 noreuse rc=$?" >> $O/status.txt
timeout 900 python bench.py --config cfg4 --geno --steps 10 --warmup 3 --no-cpu --no-e2e --opt reuse_atb=0 > $O/bench_cfg4_geno_noreuse.json 2> $O/bench_cfg4_geno_noreuse.err; echo "cfg4g noreuse rc=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1e_epilogue -s 10 -c 1 -o $O/k1e_n1e7 python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_k1e.log 2>&1
summ k1e_n1e7
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1g_aty_fused -s 10 -c 1 -o $O/k1g_cfg4 python bench.py --config cfg4 --geno --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_k1g.log 2>&1
summ k1g_cfg4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chol_d2 -s 40 -c 1 -o $O/k4_d2_cfg2 python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_d2.log 2>&1
summ k4_d2_cfg2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_sk -c 1 -o $O/k3_mxm_r10193 python tools/ncu_newton.py --r 10193 --n 20000 > $O/ncu_k3a.log 2>&1
summ k3_mxm_r10193
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_fused -c 1 -o $O/k3_smw_r435 python tools/ncu_newton.py --r 435 > $O/ncu_k3b.log 2>&1
summ k3_smw_r435
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small_cl -s 3 -c 1 -o $O/k7_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_k7.log 2>&1
summ k7_cfg1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_peer_eval -s 20 -c 1 -o $O/peer_eval_cfg2 python bench.py --config cfg2 --shard --steps 1 --warmup 3 --no-cpu --no-e2e --control host > $O/ncu_peer.log 2>&1
summ peer_eval_cfg2
du -sh $O >> $O/status.txt
echo done >> $O/status.txt
