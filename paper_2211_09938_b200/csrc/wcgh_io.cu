// C ABI: host file I/O — CGH1 holograms (image_io.cpp:220-278) and CGHL LUT
// caches (fringe_lut.cpp:95-166). No device needed.
#include "wcgh_state.cuh"

using namespace wcgh;
using namespace wcgh::abi;

extern "C" {

// ---- CGH1 files (image_io.cpp:220-278): 34-byte header + f32 payload ------

int wcgh_write_cgh1(const char* path, const float* plane, int n, const wcgh_layer* scene) {
  return guard(nullptr, [&] {
    require(path && plane && scene, "save_hologram: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "save_hologram: field size does not match scene plane_size");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw RuntimeError(std::string("hologram: cannot open ") + path + " for writing");
    const char magic[4] = {'C', 'G', 'H', '1'};
    const uint16_t version = 1;
    const uint32_t un = uint32_t(n);
    bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&version, 2, 1, f) == 1 &&
              std::fwrite(&un, 4, 1, f) == 1 && std::fwrite(&scene->wavelength, 8, 1, f) == 1 &&
              std::fwrite(&scene->pitch, 8, 1, f) == 1 && std::fwrite(&scene->z, 8, 1, f) == 1;
    const size_t count = size_t(n) * n * 2;
    ok = ok && std::fwrite(plane, sizeof(float), count, f) == count;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw RuntimeError(std::string("hologram: write failed for ") + path);
  });
}

int wcgh_read_cgh1(const char* path, float* plane, int64_t capacity, int* n_out,
                   wcgh_layer* scene_out) {
  return guard(nullptr, [&] {
    require(path != nullptr, "load_hologram: NULL path");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw RuntimeError(std::string("hologram: cannot open ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CGH1", 4) != 0)
      throw RuntimeError(std::string("hologram: bad magic in ") + path);
    uint16_t version = 0;
    uint32_t un = 0;
    wcgh_layer sc{};
    if (std::fread(&version, 2, 1, f) != 1 || std::fread(&un, 4, 1, f) != 1 ||
        std::fread(&sc.wavelength, 8, 1, f) != 1 || std::fread(&sc.pitch, 8, 1, f) != 1 ||
        std::fread(&sc.z, 8, 1, f) != 1)
      throw RuntimeError("hologram: truncated or unreadable header");
    if (version != 1) throw RuntimeError("hologram: unsupported version " + std::to_string(version));
    validate_layer(sc);
    require(un > 0 && un <= 65536 && is_pow2(int(un)),
            "scene: plane_size must be a power of two, got " + std::to_string(un));
    if (n_out) *n_out = int(un);
    if (scene_out) *scene_out = sc;
    if (plane) {
      const size_t count = size_t(un) * un;
      require(capacity >= int64_t(count), "load_hologram: output buffer too small");
      if (std::fread(plane, sizeof(float) * 2, count, f) != count)
        throw RuntimeError("hologram: truncated payload");
      for (size_t i = 0; i < 2 * count; ++i)
        if (!std::isfinite(plane[i]))
          throw ValidationError(std::string("hologram ") + path + ": non-finite sample");
    }
  });
}

// ---- CGHL LUT cache files (fringe_lut.cpp:95-166): 36-byte header + f32 ----

int wcgh_write_cghl(const char* path, const float* lut, int n, int block, const wcgh_layer* scene) {
  return guard(nullptr, [&] {
    require(path && lut && scene, "lut cache: NULL argument");
    validate_layer(*scene);
    require(is_pow2(n), "scene: plane_size must be a power of two, got " + std::to_string(n));
    require(block == 1 || block == 2 || block == 4 || block == 8,
            "build_block_lut: unsupported block size " + std::to_string(block));
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw RuntimeError(std::string("lut cache: cannot open ") + path + " for writing");
    const char magic[4] = {'C', 'G', 'H', 'L'};
    const uint16_t version = 1, b = uint16_t(block);
    const uint32_t un = uint32_t(n);
    bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&version, 2, 1, f) == 1 &&
              std::fwrite(&b, 2, 1, f) == 1 && std::fwrite(&un, 4, 1, f) == 1 &&
              std::fwrite(&scene->wavelength, 8, 1, f) == 1 &&
              std::fwrite(&scene->pitch, 8, 1, f) == 1 && std::fwrite(&scene->z, 8, 1, f) == 1;
    const size_t span = size_t(2 * n - 1);
    const size_t count = span * span * 2;
    ok = ok && std::fwrite(lut, sizeof(float), count, f) == count;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw RuntimeError(std::string("lut cache: write failed for ") + path);
  });
}

int wcgh_read_cghl(const char* path, float* lut, int64_t capacity, int* n_out, int* block_out,
                   wcgh_layer* scene_out) {
  return guard(nullptr, [&] {
    require(path != nullptr, "lut cache: NULL path");
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw RuntimeError(std::string("lut cache: cannot open ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "CGHL", 4) != 0)
      throw RuntimeError(std::string("lut cache: bad magic in ") + path);
    uint16_t version = 0, block = 0;
    uint32_t un = 0;
    wcgh_layer sc{};
    if (std::fread(&version, 2, 1, f) != 1 || std::fread(&block, 2, 1, f) != 1 ||
        std::fread(&un, 4, 1, f) != 1 || std::fread(&sc.wavelength, 8, 1, f) != 1 ||
        std::fread(&sc.pitch, 8, 1, f) != 1 || std::fread(&sc.z, 8, 1, f) != 1)
      throw RuntimeError("lut cache: truncated header");
    if (version != 1) throw RuntimeError("lut cache: unsupported version " + std::to_string(version));
    require(un > 0 && un <= 65536 && is_pow2(int(un)),
            "scene: plane_size must be a power of two, got " + std::to_string(un));
    if (n_out) *n_out = int(un);
    if (block_out) *block_out = int(block);
    if (scene_out) *scene_out = sc;
    if (lut) {
      const size_t span = size_t(2 * un - 1);
      const size_t count = span * span;
      require(capacity >= int64_t(count), "lut cache: output buffer too small");
      if (std::fread(lut, sizeof(float) * 2, count, f) != count)
        throw RuntimeError("lut cache: truncated payload");
      for (size_t i = 0; i < 2 * count; ++i)
        if (!std::isfinite(lut[i]))
          throw ValidationError(std::string("lut cache ") + path + ": non-finite sample");
    }
  });
}

}  // extern "C"

WCGH_CHK_TU(wcgh_io)
