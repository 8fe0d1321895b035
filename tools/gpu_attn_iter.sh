mkdir -p gpurun_out
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_attention_bwd.py "tests/test_gpu_train.py::test_gradient_matches_autograd" > gpurun_out/gputest_attn.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest_attn.log
