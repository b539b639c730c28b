timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/t_all.log
SG_VERBOSE=1 PRE=1 IRTS=1e-2 timeout 900 python tools/solver_experiment.py c2_4d_stream:12 > gpurun_out/solver_c2_12.log 2> gpurun_out/solver_c2_12.err
SG_OUTER=2 PRE=1 IRTS=1e-2 timeout 900 python tools/solver_experiment.py c2_4d_stream:12 c4_6d_stream:8 > gpurun_out/solver_mr.log 2>&1
PRE=1 IRTS=1e-2 timeout 900 python tools/solver_experiment.py c4_6d_stream:8 > gpurun_out/solver_c4.log 2>&1
cat gpurun_out/t_all.log
