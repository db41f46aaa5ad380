// psm_host.h — host-side helpers of the product library (voxeliser, brick packing).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace psm {

int check_mesh(const double* verts, int64_t nv, const int32_t* tris, int64_t nt,
               std::string* why);
void geometry_extent(const double* verts, int64_t nv, int s, double origin[3],
                     int64_t dims_cells[3]);
void voxelize_mesh(const double* verts, int64_t nv, const int32_t* tris, int64_t nt, int s,
                   const double origin[3], const int64_t dims_cells[3],
                   std::vector<uint8_t>& bits);
void pack_bricks(const std::vector<uint8_t>& bits, int s, const int64_t dims_cells[3],
                 std::vector<unsigned long long>& words, std::vector<uint8_t>& mask,
                 int* total_words);

}  // namespace psm
