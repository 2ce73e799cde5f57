#!/bin/bash
# One GPU call: build, full -m gpu suite (durations), then the round evidence (TAG).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build0.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/${T}_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/${T}_gputests.log
tail -30 gpurun_out/${T}_gputests.log
[ "${EVIDENCE:-1}" = "1" ] && TAG=$T bash tools/gpu_evidence.sh
