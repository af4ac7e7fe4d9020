// Tile engine compiled with 2^5 amplitudes per thread (see qsv_tile.cuh).
#define QSV_TILE_REGBITS 5
#define QSV_TILE_NS r5
#include "qsv_tile_impl.cuh"
