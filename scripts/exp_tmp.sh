# scratch: the command of the last one-off GPU experiment
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/sweep.sh "FFG_X=0"
