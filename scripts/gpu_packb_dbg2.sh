set -x
cd $GRAFT_REPO_ROOT
timeout 200 python -c "
import faulthandler, sys
faulthandler.dump_traceback_later(150, exit=True)
sys.argv = ['bench.py', '--steps', '5', '--warmup', '3', '--no-cpu-baseline']
g = {'__file__': 'bench.py', '__name__': '__main__'}; exec(compile(open('bench.py').read(), 'bench.py', 'exec'), g)
" > gpurun_out/dbg5.log 2>&1; echo "full exit $?"
