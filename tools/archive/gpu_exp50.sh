mkdir -p gpurun_out
cp paper_2603_08026_b200/csrc/attn_fused.cu /tmp/attn_new.cu
: > gpurun_out/exp50.log
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 >> gpurun_out/exp50.log
for V in new old new old; do
  if [ $V = old ]; then cp tools/_attn_old.cu paper_2603_08026_b200/csrc/attn_fused.cu; else cp /tmp/attn_new.cu paper_2603_08026_b200/csrc/attn_fused.cu; fi
  python -m paper_2603_08026_b200.build > /dev/null 2>&1
  echo "$V" >> gpurun_out/exp50.log
  timeout 300 python tools/step_gap.py --mode ro 2>&1 | head -1 >> gpurun_out/exp50.log
  timeout 300 python tools/step_gap.py --mode fi 2>&1 | head -1 >> gpurun_out/exp50.log
done
cp /tmp/attn_new.cu paper_2603_08026_b200/csrc/attn_fused.cu
