import os, sys, subprocess
for pol in ["0", "1", "2"]:
    for m in ["-2", "-4"]:
        env = dict(os.environ, FL1_LOCKSTEP_POLICY=pol, MODES=m)
        out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "batch_probe2.py")], env=env,
                             capture_output=True, text=True).stdout.splitlines()
        print("policy", pol, out[2] if len(out) > 2 else out)
