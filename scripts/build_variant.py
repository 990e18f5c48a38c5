"""Build a throwaway copy of the package under scratch/<name>/ with extra -D defines (and
optionally a replacement source file), for side-by-side timing on the GPU box via
RICI_PKG_ROOT=scratch/<name>.   python scripts/build_variant.py name "-DFOO=1" [csrc_file=path ...]"""
import os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, defines = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
d = os.path.join(ROOT, "scratch", name)
shutil.rmtree(d, ignore_errors=True)
shutil.copytree(os.path.join(ROOT, "paper_2007_02306_b200"), os.path.join(d, "paper_2007_02306_b200"),
                ignore=shutil.ignore_patterns("*.so", "__pycache__"))
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
for rep in sys.argv[3:]:
    dst, src = rep.split("=")
    shutil.copy(os.path.join(ROOT, src), os.path.join(d, "paper_2007_02306_b200", "csrc", dst))
r = subprocess.run([sys.executable, os.path.join(d, "paper_2007_02306_b200", "build.py"), "--force"],
                   env=dict(os.environ, RICI_NVCC_DEFINES=defines), capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-2000:])
print(d)
