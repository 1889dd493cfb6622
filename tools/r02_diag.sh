cd $GRAFT_REPO_ROOT
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/diag3_smi_before.txt
(nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/diag3_smi_trace.csv &) 
python tools/peel_diag.py ncf > gpurun_out/diag3.txt 2>&1
LHC_PEEL_GRID=148 python tools/peel_diag.py ncf > gpurun_out/diag3_g148.txt 2>&1
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/diag3_smi_after.txt
