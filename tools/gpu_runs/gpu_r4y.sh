mkdir -p gpurun_out
# the round-2 k_walk_bucket (TRITPERM_BATCH=0) on tables pruned by forced rows, and sticky pieces always
TRITPERM_BATCH=0 timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "c3_all or filter_list or n30 or wide_batch or ranges_and_wide or n64" > gpurun_out/r4y_batch0.log 2>&1; echo batch0=$? $(tail -1 gpurun_out/r4y_batch0.log)
TRITPERM_STICKY=2 timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "c4 or c5_window or filter_list or wide or n64 or distributed or range" > gpurun_out/r4y_sticky2.log 2>&1; echo sticky2=$? $(tail -1 gpurun_out/r4y_sticky2.log)
TRITPERM_BUCKET=0 timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "filter_list or n30" > gpurun_out/r4y_bucket0.log 2>&1; echo bucket0=$? $(tail -1 gpurun_out/r4y_bucket0.log)
