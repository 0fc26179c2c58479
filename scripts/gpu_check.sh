cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_c4.py -q -x -k "not full_batch" 2>&1 | tail -2
CFG=c4 K=20 ROLES=gemm_tU_cross,gemm_ens_qkv_attn,gemm_ens_ffn1,gemm_ens_ffn2_ln timeout 900 python scripts/dense_ab.py '[{}]' 2>&1 | tail -2
