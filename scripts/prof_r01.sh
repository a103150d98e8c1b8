set -x
python scripts/kprof.py c4 && ncu --set full --import-source on --clock-control none -k k_fast -c 1 -s 1 -o gpurun_out/prof_c4_r01c python scripts/kprof.py c4 > gpurun_out/p1.log 2>&1
python scripts/kprof.py big && ncu --set full --import-source on --clock-control none -k regex:k_fast_big -c 1 -s 1 -o gpurun_out/prof_big_r01c python scripts/kprof.py big > gpurun_out/p2.log 2>&1
python scripts/kprof_run.py c2_cdr_tanh && ncu --set full --import-source on --clock-control none -k regex:k_fast_run -c 1 -o gpurun_out/prof_run_c2 python scripts/kprof_run.py c2_cdr_tanh 200 > gpurun_out/p3.log 2>&1
python scripts/kprof_adi.py && ncu --set full --import-source on --clock-control none -k regex:k_gaptooth_exact -c 1 -s 2 -o gpurun_out/prof_adi_t1 python scripts/kprof_adi.py > gpurun_out/p4.log 2>&1
ls -la gpurun_out/*.ncu-rep | tail -4
