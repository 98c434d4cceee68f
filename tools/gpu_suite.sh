# the whole GPU suite (as the driver runs it), then the parity files again with FCT_DEBUG=1 (a synchronize and
# launch check after every kernel, hash range checks) in place of compute-sanitizer, which this pool disables
mkdir -p gpurun_out
rm -f gpurun_out/fullsize_full_data.jsonl gpurun_out/rownorm_exact_rel.jsonl
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1
echo "gpu suite rc=$? $(tail -1 gpurun_out/gputest.log)"
FCT_DEBUG=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fct2.py tests/test_gpu_coreset.py -q -m gpu -x > gpurun_out/gputest_debug.log 2>&1
echo "debug rc=$? $(tail -1 gpurun_out/gputest_debug.log)"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
