cd $GRAFT_REPO_ROOT
CFG=cfg3 python tools/host_step_profile.py
CFG=cfg2 STEPS=100 python tools/host_step_profile.py
