// Tile engine compiled with 2^4 amplitudes per thread (see qsv_tile.cuh).
#define QSV_TILE_REGBITS 4
#define QSV_TILE_NS r4
#include "qsv_tile_impl.cuh"
