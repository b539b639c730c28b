timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/t_all.log
timeout 600 python tools/step_prof.py --config c4_6d_stream > gpurun_out/sp_c4.log 2>&1
timeout 600 python tools/step_prof.py --config c2_4d_stream --L 10 > gpurun_out/sp_c2.log 2>&1
cat gpurun_out/t_all.log | tail -3
