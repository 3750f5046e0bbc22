for v in bk_m0 bk_m0f; do cp ab/$v.so paper_2502_00356_b200/libbesselgp_sm100a.so; echo "== $v"; timeout 600 python -m pytest tests -m gpu -q -x -k "besselk or bk or smoke" 2>&1 | tail -1; done
git_restore=1
bash tools/ab_libs.sh --bk ab/bk_m1.so ab/bk_m0.so ab/bk_m0f.so
