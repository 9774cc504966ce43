"""Build libairg.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2508_17517_b200.build_lib [--force]
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, 'csrc')
OBJ = os.path.join(HERE, 'build')
LIB = os.path.join(HERE, 'libairg.so')
NVCC = os.environ.get('NVCC', '/usr/local/cuda/bin/nvcc')

def _nccl_dir():
    """NCCL headers / library shipped with torch (nvidia-nccl wheel)."""
    import importlib.util
    spec = importlib.util.find_spec('nvidia')
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, 'nccl')
        if os.path.exists(os.path.join(d, 'include', 'nccl.h')):
            return d
    raise RuntimeError('nccl.h not found (nvidia-nccl wheel)')


NCCL = _nccl_dir()
FLAGS = ['-O3', '-std=c++17', '-gencode', 'arch=compute_100a,code=sm_100a', '-lineinfo',
         '-Xcompiler', '-fPIC', '--expt-relaxed-constexpr', '--extended-lambda',
         '-I', os.path.join(ROOT, 'include'), '-I', os.path.join(NCCL, 'include'),
         '-Xptxas', '-warn-spills']
LDFLAGS = ['-L', os.path.join(NCCL, 'lib'), '-l:libnccl.so.2',
           '-Xlinker', '-rpath=' + os.path.join(NCCL, 'lib')]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith('.cu'))


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith('.cuh')]
    headers.append(os.path.join(ROOT, 'include', 'airg.h'))
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + '.o')
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([NVCC] + FLAGS + ['-c', src, '-o', obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f'nvcc failed: {" ".join(cmd)}\n{r.stdout}\n{r.stderr}')
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stderr, r.stdout, file=sys.stderr)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB)
                                              for o in objs):
        cmd = [NVCC, '-shared', '-gencode', 'arch=compute_100a,code=sm_100a', '-o', LIB] + objs + LDFLAGS
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f'link failed:\n{r.stdout}\n{r.stderr}')
    return LIB


if __name__ == '__main__':
    print(build(force='--force' in sys.argv, verbose=True))
