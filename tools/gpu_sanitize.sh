# compute-sanitizer over small cases of every product kernel path (tools/sanitize_cases.py).
mkdir -p gpurun_out/san
timeout 120 python tools/sanitize_cases.py > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san/plain.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san/memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py --only z3p3,z3p4,z3p5,h3p7,s2p3,s1p4,sgq > gpurun_out/san/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san/synccheck.log
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py --only z3p3,z3p4,z3p5,h3p7,s2p3,s1p4,sgq > gpurun_out/san/initcheck.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/san/initcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py --only z3p3,z3p5,s2p3,sgq > gpurun_out/san/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san/racecheck.log
ls -la gpurun_out/san
