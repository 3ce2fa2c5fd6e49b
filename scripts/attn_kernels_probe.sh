#!/usr/bin/env bash
# K2 head_dim-128 kernels side by side on the GPU box: both-kernel parity tests,
# then scripts/micro/attn_probe.py for the mma.sync (SR_ATTN_TC=0) and tcgen05
# (SR_ATTN_TC=1) kernels on three work shapes.  Output under gpurun_out/.
timeout 300 python -m pytest tests/test_gpu_attention.py -q > gpurun_out/attn.log 2>&1; echo "rc=$?" >> gpurun_out/attn.log
: > gpurun_out/attn_probe.txt
for tc in 1 0; do for args in "" "--seqs 64 --ctx 2048 2560" "--seqs 1024 --ctx 96 200"; do
  SR_ATTN_TC=$tc timeout 120 python scripts/micro/attn_probe.py --iters 50 $args >> gpurun_out/attn_probe.txt 2>&1
  echo "tc=$tc $args" >> gpurun_out/attn_probe.txt
done; done
