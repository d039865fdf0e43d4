cd $GRAFT_REPO_ROOT
for C in 1B 70B; do echo "== $C"; timeout 300 python tools/timeline.py --config $C --steps 2 2>&1 | grep -v -i warn | tail -9; done
