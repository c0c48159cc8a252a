# C3 generation timing, twice (box-to-box comparisons use two calls on one box); TESTS=1 adds the generation parity tests
python -m paper_2206_08660_b200.build >/dev/null 2>&1 || exit 1
for i in 1 2; do timeout 300 python tools/run_pipeline.py --config ${CFG:-C3} --reps 4 2>&1 | grep -o "'${KEY:-gen}': [0-9.]*" | tr "\n" " "; echo; done
[ -n "$TESTS" ] && timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_bricked.py tests/test_gpu_c5.py 2>&1 | tail -1
true
