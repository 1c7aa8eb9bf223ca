# Same-box A/B of the GAN bench between this tree's library (A) and variant libraries (MGSR_LIB=...),
# alternating: bash tests/ab_lib.sh exp/libB.so [exp/libC.so ...]
for i in 1 2 3; do
  python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['value'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
  for v in "$@"; do
    MGSR_LIB=$v python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
  done
done
