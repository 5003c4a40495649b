# GPU: given pytest targets (default: whole -m gpu suite); summary line last
mkdir -p gpurun_out
python -m pytest ${@:-tests -m gpu} -q -x > gpurun_out/t_pytest.log 2>&1
grep -E "^E |Error|FAILED" gpurun_out/t_pytest.log | head -5
tail -1 gpurun_out/t_pytest.log
