set -x
nproc; free -g; lscpu | head -20; nvidia-smi; 
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
CP=$!
./tools/fp64_peak
kill $CP
python -c "import torch; print(torch.cuda.get_device_name(0)); import torch.distributed as d; print(hasattr(d.ProcessGroupNCCL,'_comm_ptr') if hasattr(d,'ProcessGroupNCCL') else None)"
