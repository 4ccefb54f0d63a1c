# round-2 solve evidence: launch list of one host-driven c5 solve (+ one K7 apply), and ncu --set full of
# the main per-iteration kernels (first iteration's S_T GEMV, local GEMV, coarse GEMV, phit, local2) and K7
export VB_NO_GRAPH=1
python tools/profile_solve.py --with-k7 > gpurun_out/ps_plain.log 2>&1 &&
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches_solve.csv python tools/profile_solve.py --with-k7 > gpurun_out/ps_ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"sym_gemv_kernel|phit_kernel|local2_kernel|elem_apply_bulk_kernel" -c 7 \
    -o gpurun_out/r02_solve_full python tools/profile_solve.py --with-k7 > gpurun_out/ps_ncu2.log 2>&1
ls -la gpurun_out/r02_*
