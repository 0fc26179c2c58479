cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_c4.py -q -k "tcgen05" -s 2>&1 | grep -E "attention|passed|failed|Error"
CFG=c4 K=20 ROLES=gemm_ens_qkv_attn timeout 900 python scripts/dense_ab.py '[{}, {"ens_attn_tc": 1}]' 2>&1 | tail -2
