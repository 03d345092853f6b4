set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke1.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > gpurun_out/gputest1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest1.log
