# full GPU suite + smoke (the driver's round-end tiers), logs under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ft_build.log 2>&1 || { echo build failed; tail gpurun_out/ft_build.log; exit 1; }
timeout 3300 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/ft_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/ft_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ft_smoke.log 2>&1; echo "smoke rc $?"
tail -8 gpurun_out/ft_smoke.log
