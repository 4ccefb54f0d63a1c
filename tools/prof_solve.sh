# solve evidence (TAG, default r02k): launch list of one host-driven c5 solve (+ one K7 apply), and
# ncu --set full of the main per-iteration kernels of the first iteration (K_DD^-1 GEMV of B0, local
# GEMV, phit, coarse GEMV, coarse extension, the fused local2 + entity sum, S_T GEMV, the fused
# chunk sum + gather + p.q) and K7
TAG=${TAG:-r02k}
export VB_NO_GRAPH=1
python tools/profile_solve.py --with-k7 > gpurun_out/ps_plain.log 2>&1 &&
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_solve.csv python tools/profile_solve.py --with-k7 > gpurun_out/ps_ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"sym_gemv_kernel|phit_kernel|coarse_ext_kernel|local2_entity_sum_kernel|chunk_gather_dot_kernel|cd_sum_parts_kernel|cd_interior_kernel|elem_apply_bulk_kernel" -c 14 \
    -o gpurun_out/${TAG}_solve_full python tools/profile_solve.py --with-k7 > gpurun_out/ps_ncu2.log 2>&1
# K7 (persistent pipelined element-by-element operator + its input gather), first two applications
ncu --set full --clock-control none --import-source on -k regex:"elem_apply_pipe_kernel|elem_xgather_kernel" -c 4 \
    -o gpurun_out/${TAG}_k7_full python tools/k7_time.py > gpurun_out/ps_ncu3.log 2>&1
ls -la gpurun_out/${TAG}_*
