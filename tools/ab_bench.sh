T=$1; shift
for r in 1 2; do for v in main "$@"; do
  unset DC_SO_OVERRIDE; if [ $v != main ]; then export DC_SO_OVERRIDE=$PWD/variants/libdc_$v.so; fi
  timeout 300 python -u bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 0 > gpurun_out/$T.$v.$r.log 2>&1
done; done
