// Tile engine compiled with 2^3 amplitudes per thread (see qsv_tile.cuh):
// twice the threads of r4 per tile, for small states whose passes are
// latency-bound (tiles of at most 11 qubits: 8 thread bits).
#define QSV_TILE_REGBITS 3
#define QSV_TILE_NS r3
#include "qsv_tile_impl.cuh"
