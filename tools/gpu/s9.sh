timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not config3" > gpurun_out/s9.log 2>&1; echo rc=$?
tail -5 gpurun_out/s9.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
