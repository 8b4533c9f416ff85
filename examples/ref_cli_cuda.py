"""The reference's own command line with a GPU backend registered:

    PYTHONPATH=baseline/_ref:. python -m examples.ref_cli_cuda pool --backend cuda ...

``bevpool pool / verify / bench`` (the reference's cli.py:195-243) accept
``--backend cuda`` (this package, fast mode) and ``--backend cuda_exact``
(bit-identical to the reference's interval backend) once
examples/ref_backend_cuda.register has added them to the reference's
dispatch table; the parser reads BACKENDS when it is built, so the backends
are registered first.
"""

import sys

import bevpool  # the reference
import bevpool.cli as ref_cli
import bevpool.pooling as ref_pooling

from examples.ref_backend_cuda import register

register(bevpool, "cuda")
register(bevpool, "cuda_exact", exact=True)
ref_cli.BACKENDS = ref_pooling.BACKENDS  # the CLI imported the tuple by name

if __name__ == "__main__":
    sys.exit(ref_cli.main())
