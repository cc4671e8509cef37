bash tools/gpu_round.sh s2a tests bench launches
NCU_K="k_rbgs|k_restrict|k_prolong|k_norms|k_coarse" NCU_C=30 bash tools/gpu_round.sh s2a_ref full
NCU_K="k_pass2d" NCU_C=4 bash tools/gpu_round.sh s2a_p2d full
FUSED=3 NCU_K="k_sweep3d" NCU_C=4 bash tools/gpu_round.sh s2a_s3d full
