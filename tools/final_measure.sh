#!/bin/bash
# Round-end measurements (run under gpurun --gpus 4 from the repo root): ncu capture of one steady
# split fit step, warm-L2 DRAM per step, the bench line at 1 / 2 / 4 GPUs, every config.
K="regex:^(encode_fwd|prep_image|mlp_fit|encode_bwd|adam_tma|adam)_kernel"
timeout 300 python tools/step_probe.py 3 1 > gpurun_out/sp_plain.log 2>&1 || exit 1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -s 15 -c 8 -o gpurun_out/fit_r2f python tools/step_probe.py 3 1 > gpurun_out/ncu_fit_f.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k "$K" -s 15 -c 48 --csv --log-file gpurun_out/warm_f.csv python tools/step_probe.py 3 1 > gpurun_out/ncu_warm_f.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2_bench_${n}gpu.json 2> gpurun_out/r2_bench_${n}gpu.err
done
timeout 1200 python configs.py --precision fp16,fp32 --out gpurun_out/r2_configs.json > gpurun_out/configs_final.log 2>&1
ls -la gpurun_out/fit_r2f.ncu-rep gpurun_out/warm_f.csv gpurun_out/r2_bench_*.json gpurun_out/r2_configs.json
