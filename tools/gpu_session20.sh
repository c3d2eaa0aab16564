timeout 300 ./tools/ubench_mix
timeout 600 ./tools/ubench_repulse 65428 2>&1 | grep -v COARSE
