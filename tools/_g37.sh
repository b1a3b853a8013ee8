timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g37_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/g37_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
