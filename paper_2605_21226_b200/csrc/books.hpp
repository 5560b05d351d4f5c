// books.hpp — host codebook registry (product side; see books.cpp).
#pragma once
#include <array>
#include <cstdint>
#include <vector>

namespace oqh {

struct Book {
  int bits = 0;
  double lo = 0.0, hi = 0.0;
  std::vector<double> centroids;   // ascending, 2^bits
  std::vector<double> boundaries;  // midpoints, 2^bits - 1
};

const Book& xi_book(int bits);                // books.hpp:69-74
const Book& rho_book(uint32_t d, int bits);   // books.hpp:86-95
Book custom_book(const double* centroids, int bits);  // Books::custom (codec.hpp:134-140)
std::array<double, 2> oct_encode(const double n[3]);
std::array<double, 3> oct_decode(double xi, double eta);
uint64_t rotation_sign_mask_word(uint64_t seed, uint32_t i);

}  // namespace oqh
