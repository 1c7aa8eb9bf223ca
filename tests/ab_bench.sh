# Same-box A/B of the GAN bench: A = the tree in exp/abA (a git worktree of an older commit, built in place),
# B = this tree, alternating.  Not part of the product; used to compare kernel variants on one GPU.
for i in 1 2 3; do
  (cd exp/abA && python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['value'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])")
  python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['value'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
done
