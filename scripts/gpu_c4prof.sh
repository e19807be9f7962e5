cd $GRAFT_REPO_ROOT
timeout 300 python scripts/c4_local_profile.py 2 > gpurun_out/c4prof.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/c4_launches.csv python scripts/c4_local_profile.py 2 > gpurun_out/c4ncu.log 2>&1; echo rc=$?
