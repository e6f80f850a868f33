# Pipeline trace of CTA 0 (debug): build the trace variant first with
#   scripts/build_variants.sh tr:"-DBSA_TC_TRACE_BUILD"
# then run this under gpurun and analyse with scripts/trace_analyze.py.
mkdir -p gpurun_out
BSA_LIB_VARIANT=tr BSA_TC_TRACE=gpurun_out/trace200.bin timeout -s KILL 200 python scripts/profile_step.py --steps 1 > gpurun_out/trace.log 2>&1
