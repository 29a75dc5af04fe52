cd $GRAFT_REPO_ROOT
for cfg in "1 148 8" "2 148 8" "4 148 8" "2 148 12" "4 148 12" "8 144 8"; do timeout 60 ./tools/tma_mcast_probe $cfg; done
